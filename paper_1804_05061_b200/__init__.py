"""B200-native SRWCR hot path (arXiv 1804.05061): thin Python binding of libsrwcr.so.

This module only marshals arguments to the C ABI declared in ``include/srwcr.h``;
every step of the evaluation runs in the sm_100a kernels of ``csrc/``.  There is no
CPU fallback: importing works without a GPU, but creating a context fails loudly if
the library or a CUDA device is missing.

Arrays may be numpy arrays (host) or torch tensors (host or CUDA); device tensors
are passed as device pointers (the fast path).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_ROOT = os.path.dirname(_HERE)
_LIB = os.environ.get("SRWCR_LIB") or os.path.join(_HERE, "libsrwcr.so")   # (SRWCR_LIB: another build of csrc/, experiments)
_SRCS = [os.path.join(_HERE, "csrc", f) for f in ("srwcr.cu", "srwcr_kernels.cuh", "srwcr_fast.cuh", "srwcr_register.inc",
                                                  "srwcr_fields.inc")]
_HDR = os.path.join(_ROOT, "include", "srwcr.h")

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared"]

# status codes (include/srwcr.h)
OK, EINVAL, ENOMEM, ECUDA, ENCCL, EDEGENERATE, ENOTSUP, ESTATE, ENONFINITE = 0, -1, -2, -3, -4, -5, -6, -7, -8
DUMP = dict(fixed=1, moving=2, a0=3, ctrl_taps=4, spat_taps=5, N=6, SQ=7, regions=8, coefs=9, warped=10)


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile csrc/ into libsrwcr.so in-tree with nvcc for sm_100a."""
    newest = max(os.path.getmtime(p) for p in _SRCS + [_HDR])
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < newest:
        nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
        tmp = _LIB + f".tmp{os.getpid()}"
        cmd = [nvcc, *NVCC_FLAGS, *(["-Xptxas", "-v"] if verbose else []), "-o", tmp, _SRCS[0], "-ldl"]
        subprocess.check_call(cmd)
        os.replace(tmp, _LIB)
    return _LIB


class SrwcrError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"srwcr status {status}: {msg}")
        self.status = status


class _Options(ctypes.Structure):
    _fields_ = [("struct_size", ctypes.c_int32), ("orientation", ctypes.c_int32),
                ("inputs_normalized", ctypes.c_int32), ("device", ctypes.c_int32),
                ("nranks", ctypes.c_int32), ("rank", ctypes.c_int32), ("nccl_id", ctypes.c_void_p),
                ("eps_mass", ctypes.c_double), ("eps_sigma", ctypes.c_double),
                ("moment_shift", ctypes.c_int32), ("use_graph", ctypes.c_int32), ("grad_exchange", ctypes.c_int32)]


class _Stats(ctypes.Structure):
    _fields_ = [("launches_total", ctypes.c_int64), ("launches_per_eval", ctypes.c_int32),
                ("ms_pass1", ctypes.c_float), ("ms_combine", ctypes.c_float), ("ms_pass2", ctypes.c_float),
                ("ms_total", ctypes.c_float), ("warps_per_cta", ctypes.c_int32), ("slot_capacity", ctypes.c_int32),
                ("voxels_per_lane", ctypes.c_int32), ("items", ctypes.c_int32), ("ms_prep", ctypes.c_float),
                ("warps_per_cta2", ctypes.c_int32), ("items2", ctypes.c_int32),
                ("exact_voxels", ctypes.c_int32), ("exact_capacity", ctypes.c_int32),
                ("pipe_items1", ctypes.c_int32), ("pipe_items2", ctypes.c_int32),
                ("fast_path", ctypes.c_int32), ("fast_items", ctypes.c_int32), ("fast_warps", ctypes.c_int32),
                ("fast_slots", ctypes.c_int32)]


class _LbfgsConfig(ctypes.Structure):
    _fields_ = [("struct_size", ctypes.c_int32), ("m", ctypes.c_int32), ("max_iter", ctypes.c_int32),
                ("max_linesearch", ctypes.c_int32), ("w_p", ctypes.c_double), ("ftol", ctypes.c_double),
                ("wolfe", ctypes.c_double), ("stable_window", ctypes.c_int32), ("verbose", ctypes.c_int32),
                ("stable_tol", ctypes.c_double), ("epsilon", ctypes.c_double)]


class _Report(ctypes.Structure):
    _fields_ = [("struct_size", ctypes.c_int32), ("iterations", ctypes.c_int32), ("evaluations", ctypes.c_int32),
                ("status", ctypes.c_int32), ("gradient_evaluations", ctypes.c_int32),
                ("initial_cost", ctypes.c_double), ("final_cost", ctypes.c_double),
                ("final_value", ctypes.c_double), ("final_penalty", ctypes.c_double),
                ("grad_norm", ctypes.c_double)]


REGISTER_STATUS = {0: "converged", 1: "stable", 2: "max_iter", 3: "line_search_failed"}

_lib = None

EXPORTS = ["srwcr_default_options", "srwcr_create", "srwcr_num_params", "srwcr_eval", "srwcr_eval_begin",
           "srwcr_stats_buffer", "srwcr_eval_end", "srwcr_plan_slab", "srwcr_plan_layers", "srwcr_grad_layers",
           "srwcr_default_lbfgs_config",
           "srwcr_register", "srwcr_bending", "srwcr_field", "srwcr_resample", "srwcr_compose",
           "srwcr_downsample2", "srwcr_upsample2_field", "srwcr_debug_size", "srwcr_debug_dump", "srwcr_set_timing", "srwcr_get_stats",
           "srwcr_stream", "srwcr_last_error", "srwcr_destroy"]


def lib():
    """The loaded libsrwcr.so (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            raise RuntimeError(f"{_LIB} is missing: run paper_1804_05061_b200.build() (nvcc, sm_100a)")
        L = ctypes.CDLL(_LIB)
        vp, i32, i64, dbl = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
        P = ctypes.POINTER
        L.srwcr_default_options.argtypes = [P(_Options)]
        L.srwcr_create.argtypes = [P(vp), vp, vp, P(i64), P(dbl), i32, P(i32), P(dbl), P(_Options)]
        L.srwcr_num_params.argtypes = [vp, P(i64), P(i64)]
        L.srwcr_eval.argtypes = [vp, vp, P(dbl), vp]
        L.srwcr_eval_begin.argtypes = [vp, vp]
        L.srwcr_stats_buffer.argtypes = [vp, P(vp), P(ctypes.c_size_t)]
        L.srwcr_eval_end.argtypes = [vp, P(dbl), vp]
        L.srwcr_plan_slab.argtypes = [i64, i32, i32, P(i64), P(i64)]
        L.srwcr_plan_layers.argtypes = [i64, i32, i32, P(i32), i64, P(i64)]
        L.srwcr_grad_layers.argtypes = [vp, P(i64)]
        L.srwcr_debug_size.argtypes = [vp, i32, P(ctypes.c_size_t)]
        L.srwcr_debug_dump.argtypes = [vp, i32, vp, ctypes.c_size_t]
        L.srwcr_set_timing.argtypes = [vp, i32]
        L.srwcr_get_stats.argtypes = [vp, P(_Stats)]
        L.srwcr_stream.argtypes = [vp, P(vp)]
        L.srwcr_last_error.argtypes = [vp]
        L.srwcr_last_error.restype = ctypes.c_char_p
        L.srwcr_destroy.argtypes = [vp]
        L.srwcr_register.argtypes = [vp, vp, P(_LbfgsConfig), P(_Report)]
        L.srwcr_default_lbfgs_config.argtypes = [P(_LbfgsConfig)]
        L.srwcr_bending.argtypes = [vp, vp, P(dbl), vp]
        L.srwcr_field.argtypes = [vp, vp, vp]
        L.srwcr_resample.argtypes = [vp, P(i64), vp, vp, vp]
        L.srwcr_compose.argtypes = [vp, vp, P(i64), vp, vp]
        L.srwcr_downsample2.argtypes = [vp, P(i64), vp, vp]
        L.srwcr_upsample2_field.argtypes = [vp, P(i64), vp, P(i64), vp]
        for name in EXPORTS:
            if name not in ("srwcr_last_error", "srwcr_destroy"):
                getattr(L, name).restype = ctypes.c_int
        _lib = L
    return _lib


def plan_slab(nz: int, nranks: int, rank: int):
    """z-slab [z0, z1) of `rank` (host-only C function of the library)."""
    z0, z1 = ctypes.c_int64(), ctypes.c_int64()
    st = lib().srwcr_plan_slab(int(nz), int(nranks), int(rank), ctypes.byref(z0), ctypes.byref(z1))
    if st != OK:
        raise SrwcrError(st, "plan_slab")
    return z0.value, z1.value


def plan_layers(nz: int, nranks: int, rank: int, cbz, gz: int):
    """Node-layer plan of `rank`'s gradient (host-only C function): (t0, t1, o0, o1, r1) --
    touched layers [t0, t1), owned layers [o0, o1), rank - 1's partial on [o0, r1); the rank
    sends [o1, t1) to rank + 1.  cbz: tap base of every slice (int32, length nz)."""
    cb = np.ascontiguousarray(cbz, dtype=np.int32)
    if cb.size != int(nz):
        raise ValueError("cbz must have nz entries")
    out = (ctypes.c_int64 * 5)()
    st = lib().srwcr_plan_layers(int(nz), int(nranks), int(rank), cb.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                                 int(gz), out)
    if st != OK:
        raise SrwcrError(st, "plan_layers")
    return tuple(out)


def _ptr(a, n=None, what="array", out=False):
    """(pointer, keepalive) of a contiguous numpy array or torch tensor.  With n it must be
    float64 with n elements (params / gradient: the library reads or writes n doubles);
    an input is made contiguous by a copy, an output (out=True) must already be."""
    if a is None:
        return None, None
    if hasattr(a, "data_ptr"):          # torch tensor
        if n is not None:
            import torch
            if a.dtype != torch.float64 or a.numel() != n:
                raise ValueError(f"{what}: need a float64 tensor of {n} elements, got {a.dtype} x {a.numel()}")
        if not a.is_contiguous():
            if out:
                raise ValueError(f"{what}: output tensor must be contiguous")
            a = a.contiguous()
        return ctypes.c_void_p(a.data_ptr()), a
    if n is not None and (a.dtype != np.float64 or a.size != n):
        raise ValueError(f"{what}: need a float64 array of {n} elements, got {a.dtype} x {a.size}")
    if not a.flags["C_CONTIGUOUS"]:
        if out:
            raise ValueError(f"{what}: output array must be C-contiguous")
        a = np.ascontiguousarray(a)
    return a.ctypes.data_as(ctypes.c_void_p), a


class Srwcr:
    """One SRWCR problem on one GPU (or one rank of a z-slab decomposition).

    fixed, moving: float32 [Nz, Ny, Nx] (numpy or torch, host or device), raw
    intensities (normalised to [0, bins-1] by the library) unless
    inputs_normalized.  spacing_mm, control_spacing_mm: per axis (x, y, z).
    spatial_bins: k cells per axis (x, y, z); 0 = one region on that axis.
    """

    def __init__(self, fixed, moving, spacing_mm, bins, spatial_bins, control_spacing_mm, *,
                 inputs_normalized=False, device=0, nranks=1, rank=0, nccl_id=None, eps_mass=1e-12,
                 eps_sigma=1e-6, moment_shift=True, use_graph=True, orientation=0, grad_exchange=0):
        L = lib()
        shape = tuple(int(s) for s in fixed.shape)
        if tuple(moving.shape) != shape or len(shape) != 3:
            raise ValueError("fixed and moving must both be [Nz, Ny, Nx]")
        self.dims = (shape[2], shape[1], shape[0])
        opt = _Options()
        L.srwcr_default_options(ctypes.byref(opt))
        opt.inputs_normalized = int(bool(inputs_normalized))
        opt.orientation = int(orientation)
        opt.device = int(device)
        opt.nranks, opt.rank = int(nranks), int(rank)
        self._nccl_id = None
        if nccl_id is not None:
            self._nccl_id = ctypes.create_string_buffer(bytes(nccl_id), 128)
            opt.nccl_id = ctypes.cast(self._nccl_id, ctypes.c_void_p)
        opt.eps_mass, opt.eps_sigma = float(eps_mass), float(eps_sigma)
        opt.moment_shift, opt.use_graph = int(bool(moment_shift)), int(bool(use_graph))
        opt.grad_exchange = int(grad_exchange)
        fp, fk = _ptr(fixed if hasattr(fixed, "data_ptr") else np.asarray(fixed, dtype=np.float32))
        mp, mk = _ptr(moving if hasattr(moving, "data_ptr") else np.asarray(moving, dtype=np.float32))
        dims = (ctypes.c_int64 * 3)(*self.dims)
        sp = (ctypes.c_double * 3)(*map(float, spacing_mm))
        sb = (ctypes.c_int32 * 3)(*map(int, spatial_bins))
        cs = (ctypes.c_double * 3)(*map(float, control_spacing_mm))
        self._ctx = ctypes.c_void_p()
        st = L.srwcr_create(ctypes.byref(self._ctx), fp, mp, dims, sp, int(bins), sb, cs, ctypes.byref(opt))
        if st != OK:
            msg = self.last_error()
            self.close()
            raise SrwcrError(st, msg)
        n = ctypes.c_int64()
        gd = (ctypes.c_int64 * 3)()
        L.srwcr_num_params(self._ctx, ctypes.byref(n), gd)
        self.nparams = n.value
        self.grid = tuple(gd)                       # (Gx, Gy, Gz)
        self.ndim = 2 if self.dims[2] == 1 else 3
        self.params_shape = (self.ndim, self.grid[2], self.grid[1], self.grid[0])
        self._nparams = int(np.prod(self.params_shape))
        self.bins = int(bins)

    # -- core
    def last_error(self) -> str:
        return lib().srwcr_last_error(self._ctx).decode() if self._ctx else ""

    def _check(self, st):
        if st != OK:
            raise SrwcrError(st, self.last_error())

    def eval(self, params, grad=None, want_grad=True):
        """D and dD/dPhi at params ([ndim, Gz, Gy, Gx] float64, numpy or torch).

        grad: optional preallocated output (numpy or torch, host or device); by default a
        numpy array is returned when want_grad.  Returns (D, grad or None)."""
        n = self._nparams
        pp, pk = _ptr(params if hasattr(params, "data_ptr") else np.ascontiguousarray(params, dtype=np.float64), n, "params")
        if want_grad and grad is None:
            grad = np.empty(self.params_shape, dtype=np.float64)
        gp, gk = _ptr(grad, n, "grad", out=True) if want_grad else (None, None)
        self._order_after_caller(pk, gk)
        D = ctypes.c_double()
        st = lib().srwcr_eval(self._ctx, pp, ctypes.byref(D), gp)
        self._check(st)
        return D.value, (grad if want_grad else None)

    def _order_after_caller(self, *tensors):
        """The library works on its own stream: when params / grad are CUDA tensors, order it
        after torch's current stream (pending writes of params, reads of an earlier grad).  The
        call returns after its stream has finished, so later torch work is ordered too."""
        if not any(getattr(t, "is_cuda", False) for t in tensors):
            return
        import torch
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream())
        torch.cuda.ExternalStream(self.stream_handle()).wait_event(ev)

    def eval_begin(self, params):
        pp, pk = _ptr(params if hasattr(params, "data_ptr") else np.ascontiguousarray(params, dtype=np.float64),
                      self._nparams, "params")
        self._order_after_caller(pk)
        self._check(lib().srwcr_eval_begin(self._ctx, pp))

    def stats_buffer(self):
        """(device pointer, count) of the rank-partial fp64 statistics."""
        p, n = ctypes.c_void_p(), ctypes.c_size_t()
        self._check(lib().srwcr_stats_buffer(self._ctx, ctypes.byref(p), ctypes.byref(n)))
        return p.value, n.value

    def eval_end(self, grad=None, want_grad=True):
        if want_grad and grad is None:
            grad = np.empty(self.params_shape, dtype=np.float64)
        gp, gk = _ptr(grad, self._nparams, "grad", out=True) if want_grad else (None, None)
        D = ctypes.c_double()
        self._check(lib().srwcr_eval_end(self._ctx, ctypes.byref(D), gp))
        return D.value, (grad if want_grad else None)

    def bending(self, params, grad=None, want_grad=True):
        """(C_p, dC_p/dPhi): bending energy of the FFD (Eq 1; reading c19)."""
        n = self._nparams
        pp, pk = _ptr(params if hasattr(params, "data_ptr") else np.ascontiguousarray(params, dtype=np.float64), n, "params")
        if want_grad and grad is None:
            grad = np.empty(self.params_shape, dtype=np.float64)
        gp, gk = _ptr(grad, n, "grad", out=True) if want_grad else (None, None)
        E = ctypes.c_double()
        self._check(lib().srwcr_bending(self._ctx, pp, ctypes.byref(E), gp))
        return E.value, (grad if want_grad else None)

    def register(self, params=None, **cfg):
        """L-BFGS minimisation of C = D + w_p C_p (Eq 1) from params (default 0).

        cfg: any field of srwcr_lbfgs_config (m, max_iter, max_linesearch, w_p, ftol,
        wolfe, stable_window, verbose, stable_tol, epsilon).  Returns (params, report)."""
        c = _LbfgsConfig()
        lib().srwcr_default_lbfgs_config(ctypes.byref(c))
        for k, v in cfg.items():
            if k not in dict(_LbfgsConfig._fields_) or k == "struct_size":
                raise TypeError(f"unknown L-BFGS option {k}")
            setattr(c, k, v)
        x = np.zeros(self.params_shape) if params is None else np.array(params, dtype=np.float64, copy=True)
        x = np.ascontiguousarray(x)
        if x.size != self._nparams:
            raise ValueError(f"params: need {self._nparams} elements, got {x.size}")
        rep = _Report()
        rep.struct_size = ctypes.sizeof(_Report)
        self._check(lib().srwcr_register(self._ctx, x.ctypes.data_as(ctypes.c_void_p), ctypes.byref(c),
                                         ctypes.byref(rep)))
        out = {f: getattr(rep, f) for f, _ in _Report._fields_ if f != "struct_size"}
        out["status_name"] = REGISTER_STATUS.get(rep.status, "?")
        return x, out

    def field(self, params, out=None):
        """Dense FFD displacement field u(x), float32 [3, Nz, Ny, Nx] (numpy, or `out`)."""
        pp, pk = _ptr(params if hasattr(params, "data_ptr") else np.ascontiguousarray(params, dtype=np.float64),
                      self._nparams, "params")
        if out is None:
            out = np.empty((3, self.dims[2], self.dims[1], self.dims[0]), dtype=np.float32)
        nv = 3 * self.dims[0] * self.dims[1] * self.dims[2]
        if (out.numel() if hasattr(out, "numel") else out.size) != nv or str(out.dtype).split(".")[-1] != "float32":
            raise ValueError(f"out: need a float32 buffer of {nv} elements")
        op, ok_ = _ptr(out, out=True)
        self._check(lib().srwcr_field(self._ctx, pp, op))
        return out

    def debug_dump(self, what: str) -> np.ndarray:
        code = DUMP[what]
        n = ctypes.c_size_t()
        self._check(lib().srwcr_debug_size(self._ctx, code, ctypes.byref(n)))
        dtype = {"fixed": np.float32, "moving": np.float32, "a0": np.int16, "ctrl_taps": np.int32,
                 "spat_taps": np.int32, "coefs": np.float32, "warped": np.float32}.get(what, np.float64)
        out = np.empty(n.value // np.dtype(dtype).itemsize, dtype=dtype)
        self._check(lib().srwcr_debug_dump(self._ctx, code, out.ctypes.data_as(ctypes.c_void_p), n.value))
        return out

    def set_timing(self, on=True):
        self._check(lib().srwcr_set_timing(self._ctx, int(bool(on))))

    def stats(self) -> dict:
        s = _Stats()
        self._check(lib().srwcr_get_stats(self._ctx, ctypes.byref(s)))
        return {f: getattr(s, f) for f, _ in _Stats._fields_}

    def grad_layers(self):
        """plan_layers of this context's rank: (t0, t1, o0, o1, r1)."""
        out = (ctypes.c_int64 * 5)()
        self._check(lib().srwcr_grad_layers(self._ctx, out))
        return tuple(out)

    def stream_handle(self) -> int:
        p = ctypes.c_void_p()
        self._check(lib().srwcr_stream(self._ctx, ctypes.byref(p)))
        return p.value or 0

    def close(self):
        if getattr(self, "_ctx", None) and self._ctx.value:
            lib().srwcr_destroy(self._ctx)
            self._ctx = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


# ---------------------------------------------------------------- field utilities (row F4)
def _dims_arr(shape):
    nz, ny, nx = (int(s) for s in shape[-3:])
    return (ctypes.c_int64 * 3)(nx, ny, nz)


def _dev(t):
    if not (hasattr(t, "is_cuda") and t.is_cuda and t.is_contiguous()):
        raise ValueError("device (CUDA) contiguous tensors required")
    return ctypes.c_void_p(t.data_ptr())


def _stream():
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def resample(vol, field, out=None):
    """out(x) = vol(x + u(x)) (trilinear, clamped); vol [Nz,Ny,Nx], field [3,Nz,Ny,Nx] fp32 CUDA tensors."""
    import torch
    out = torch.empty_like(vol) if out is None else out
    st = lib().srwcr_resample(_dev(vol), _dims_arr(vol.shape), _dev(field), _dev(out), _stream())
    if st != OK:
        raise SrwcrError(st, "srwcr_resample")
    return out


def compose(U, u, out=None):
    """Field of 'warp by u, then by U': out(x) = u(x) + U(x + u(x))."""
    import torch
    out = torch.empty_like(u) if out is None else out
    st = lib().srwcr_compose(_dev(U), _dev(u), _dims_arr(u.shape), _dev(out), _stream())
    if st != OK:
        raise SrwcrError(st, "srwcr_compose")
    return out


def downsample2(vol):
    """2x pyramid level of an fp32 CUDA volume [Nz,Ny,Nx] (a 1-slice z axis stays 1)."""
    import torch
    nz, ny, nx = vol.shape
    out = torch.empty(((nz + 1) // 2 if nz > 1 else 1, (ny + 1) // 2, (nx + 1) // 2), dtype=vol.dtype, device=vol.device)
    st = lib().srwcr_downsample2(_dev(vol), _dims_arr(vol.shape), _dev(out), _stream())
    if st != OK:
        raise SrwcrError(st, "srwcr_downsample2")
    return out


def upsample2_field(coarse, fine_shape):
    """Fine field [3, *fine_shape] from a coarse one (values doubled: voxel units)."""
    import torch
    out = torch.empty((3, *fine_shape), dtype=coarse.dtype, device=coarse.device)
    st = lib().srwcr_upsample2_field(_dev(coarse), _dims_arr(coarse.shape), _dev(out), _dims_arr(fine_shape), _stream())
    if st != OK:
        raise SrwcrError(st, "srwcr_upsample2_field")
    return out
