"""B200-native fast tensor-vector product / multi-marginal Sinkhorn, L1 cost (arXiv 2405.19246).

Thin Python binding of ``libmmot.so`` (C ABI in ``include/mmot.h``).  Argument
marshalling only: every step of the path runs in the library's CUDA kernels.
PyTorch is used for device memory and streams.  There is no CPU fallback: if
the shared library is missing or no CUDA device is present the calls raise.
"""
from __future__ import annotations

import ctypes
import math
import os
from typing import List, Optional, Sequence

__all__ = ["Context", "VirtualGroup", "MMOTError", "lib_path", "load_library", "STATUS", "exported_symbols", "nccl_unique_id",
           "shard_range", "compose_rank_carries", "compose_rank_affine"]

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libmmot.so")
_lib = None

STATUS = {
    0: "MMOT_OK", 1: "MMOT_EINVAL", 2: "MMOT_ESHAPE", 3: "MMOT_ENONFINITE", 4: "MMOT_ENEGMASS",
    5: "MMOT_EZEROMASS", 6: "MMOT_EOVERFLOW", 7: "MMOT_ECUDA", 8: "MMOT_ENCCL", 9: "MMOT_ENOMEM",
    10: "MMOT_EUNSUPPORTED", 11: "MMOT_EPRECISION",
}

F64, F32 = 0, 1
LOG, LINEAR = 0, 1


class MMOTError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status
        self.name = STATUS.get(status, str(status))


class _Grid(ctypes.Structure):
    _fields_ = [("x_min", ctypes.c_double), ("x_max", ctypes.c_double)]


class _Grid2d(ctypes.Structure):
    _fields_ = [("x_min", ctypes.c_double), ("x_max", ctypes.c_double), ("y_min", ctypes.c_double),
                ("y_max", ctypes.c_double)]


class _Opts(ctypes.Structure):
    _fields_ = [("check_every", ctypes.c_int), ("residual_mode", ctypes.c_int),
                ("repr", ctypes.c_int), ("chunk", ctypes.c_int), ("kernel", ctypes.c_int)]


class _Report(ctypes.Structure):
    _fields_ = [("iters_done", ctypes.c_int), ("residual", ctypes.c_double), ("converged", ctypes.c_int),
                ("status", ctypes.c_int), ("fail_iter", ctypes.c_int)]


def lib_path() -> str:
    return _LIB_PATH


def load_library():
    """Load libmmot.so (fails loudly if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise ImportError(f"{_LIB_PATH} not built; run `python -m paper_2405_19246_b200._build` "
                          "or __graft_entry__.build()")
    lib = ctypes.CDLL(_LIB_PATH)
    vp = ctypes.c_void_p
    vpp = ctypes.POINTER(ctypes.c_void_p)
    lib.mmot_create.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_double, _Grid, ctypes.c_int,
                                ctypes.POINTER(_Opts), vp, ctypes.POINTER(vp)]
    lib.mmot_create.restype = ctypes.c_int
    lib.mmot_create_batched.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.POINTER(ctypes.c_double),
                                        _Grid, ctypes.c_int, ctypes.POINTER(_Opts), vp, ctypes.POINTER(vp)]
    lib.mmot_create_batched.restype = ctypes.c_int
    lib.mmot_create_2d.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.c_double, _Grid2d, ctypes.c_int,
                                   ctypes.POINTER(_Opts), vp, ctypes.POINTER(vp)]
    lib.mmot_create_2d.restype = ctypes.c_int
    lib.mmot_create_points.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_double, ctypes.POINTER(ctypes.c_double),
                                       ctypes.c_int, ctypes.POINTER(_Opts), vp, ctypes.POINTER(vp)]
    lib.mmot_create_points.restype = ctypes.c_int
    lib.mmot_create_batched_points.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.POINTER(ctypes.c_double),
                                               ctypes.POINTER(ctypes.c_double), ctypes.c_int, ctypes.POINTER(_Opts), vp,
                                               ctypes.POINTER(vp)]
    lib.mmot_create_batched_points.restype = ctypes.c_int
    lib.mmot_create_sharded.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_double, _Grid, ctypes.c_int, vp,
                                        ctypes.c_int, ctypes.c_int, ctypes.POINTER(_Opts), vp, ctypes.POINTER(vp)]
    lib.mmot_create_sharded.restype = ctypes.c_int
    lib.mmot_create_sharded_virtual.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_double, _Grid, ctypes.c_int,
                                                vp, ctypes.c_int, ctypes.POINTER(_Opts), vp, ctypes.POINTER(vp)]
    lib.mmot_create_sharded_virtual.restype = ctypes.c_int
    lib.mmot_vgroup_create.argtypes = [ctypes.c_int, ctypes.POINTER(vp)]
    lib.mmot_vgroup_create.restype = ctypes.c_int
    lib.mmot_vgroup_destroy.argtypes = [vp]
    lib.mmot_vgroup_destroy.restype = None
    lib.mmot_nccl_unique_id.argtypes = [vp]
    lib.mmot_nccl_unique_id.restype = ctypes.c_int
    lib.mmot_shard_range.argtypes = [ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int64),
                                     ctypes.POINTER(ctypes.c_int64)]
    lib.mmot_shard_range.restype = None
    dpp = ctypes.POINTER(ctypes.c_double)
    lib.mmot_compose_rank_carries.argtypes = [ctypes.c_int, dpp, ctypes.c_int, ctypes.c_int, dpp, dpp]
    lib.mmot_compose_rank_carries.restype = ctypes.c_int
    lib.mmot_compose_rank_affine.argtypes = [ctypes.c_int, dpp, ctypes.c_int, ctypes.c_int, dpp, dpp]
    lib.mmot_compose_rank_affine.restype = ctypes.c_int
    lib.mmot_marginal.argtypes = [vp, ctypes.c_int, vpp, vp]
    lib.mmot_marginal.restype = ctypes.c_int
    lib.mmot_sinkhorn.argtypes = [vp, vpp, ctypes.c_int, ctypes.c_double, vpp, ctypes.POINTER(_Report)]
    lib.mmot_sinkhorn.restype = ctypes.c_int
    lib.mmot_sinkhorn_host.argtypes = [vp, vpp, ctypes.c_int, ctypes.c_double, vpp, ctypes.POINTER(_Report)]
    lib.mmot_sinkhorn_host.restype = ctypes.c_int
    lib.mmot_cost.argtypes = [vp, vpp, ctypes.POINTER(ctypes.c_double)]
    lib.mmot_cost.restype = ctypes.c_int
    lib.mmot_cost_staged.argtypes = [vp, ctypes.POINTER(ctypes.c_double)]
    lib.mmot_cost_staged.restype = ctypes.c_int
    lib.mmot_init_uniform.argtypes = [vp, vpp]
    lib.mmot_init_uniform.restype = ctypes.c_int
    lib.mmot_destroy.argtypes = [vp]
    lib.mmot_destroy.restype = None
    lib.mmot_strerror.argtypes = [ctypes.c_int]
    lib.mmot_strerror.restype = ctypes.c_char_p
    lib.mmot_last_error.argtypes = [vp]
    lib.mmot_last_error.restype = ctypes.c_char_p
    lib.mmot_version.argtypes = []
    lib.mmot_version.restype = ctypes.c_int
    lib.mmot_info.argtypes = [vp, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64),
                              ctypes.POINTER(ctypes.c_int)]
    lib.mmot_info.restype = ctypes.c_int
    lib.mmot_launch_count.argtypes = [vp]
    lib.mmot_launch_count.restype = ctypes.c_int64
    lib.mmot_fallback_count.argtypes = [vp]
    lib.mmot_fallback_count.restype = ctypes.c_int64
    lib.mmot_stable_fallback_count.argtypes = [vp]
    lib.mmot_stable_fallback_count.restype = ctypes.c_int64
    lib.mmot_allres_checks.argtypes = [vp]
    lib.mmot_allres_checks.restype = ctypes.c_int64
    lib.mmot_graph_solves.argtypes = [vp]
    lib.mmot_graph_solves.restype = ctypes.c_int64
    lib.mmot_pair_solves.argtypes = [vp]
    lib.mmot_pair_solves.restype = ctypes.c_int64
    lib.mmot_pair_f32_solves.argtypes = [vp]
    lib.mmot_pair_f32_solves.restype = ctypes.c_int64
    lib.mmot_pair_redo_count.argtypes = [vp]
    lib.mmot_pair_redo_count.restype = ctypes.c_int64
    lib.mmot_cta_solves.argtypes = [vp]
    lib.mmot_cta_solves.restype = ctypes.c_int64
    lib.mmot_profile_enable.argtypes = [vp, ctypes.c_int]
    lib.mmot_profile_enable.restype = ctypes.c_int
    dp = ctypes.POINTER(ctypes.c_double)
    lib.mmot_profile_read.argtypes = [vp, dp, dp, ctypes.POINTER(ctypes.c_int64)]
    lib.mmot_profile_read.restype = ctypes.c_int
    _lib = lib
    return lib


def exported_symbols() -> List[str]:
    """Dynamic symbols of libmmot.so starting with ``mmot_`` (no GPU needed)."""
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", _LIB_PATH], capture_output=True, text=True, check=True).stdout
    return sorted({ln.split()[-1] for ln in out.splitlines() if ln.split() and ln.split()[-1].startswith("mmot_")})


def _ptr_array(ptrs: Sequence[int]):
    arr = (ctypes.c_void_p * len(ptrs))()
    for i, p in enumerate(ptrs):
        arr[i] = p
    return arr


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id for a sharded context (create on one rank, broadcast)."""
    lib = load_library()
    buf = ctypes.create_string_buffer(128)
    st = lib.mmot_nccl_unique_id(buf)
    if st != 0:
        raise MMOTError(st, lib.mmot_last_error(None).decode())
    return buf.raw


def shard_range(N_global: int, rank: int, world: int):
    """Grid chunk [lo, hi) owned by `rank` (host logic of the C ABI, no GPU needed)."""
    lib = load_library()
    lo, hi = ctypes.c_int64(), ctypes.c_int64()
    lib.mmot_shard_range(int(N_global), int(rank), int(world), ctypes.byref(lo), ctypes.byref(hi))
    return lo.value, hi.value


def compose_rank_carries(l: int, ops_all, world: int, rank: int):
    """Host reference of the sharded carry composition (C ABI, no GPU needed).
    ops_all: float64 array [world][2][l * 2**(l-1)].  Returns (fin, bin) arrays of 2**(l-1)."""
    import numpy as np
    lib = load_library()
    a = np.ascontiguousarray(ops_all, dtype=np.float64)
    M = 1 << (l - 1)
    fin, bin_ = np.zeros(M), np.zeros(M)
    dp = ctypes.POINTER(ctypes.c_double)
    st = lib.mmot_compose_rank_carries(int(l), a.ctypes.data_as(dp), int(world), int(rank), fin.ctypes.data_as(dp),
                                       bin_.ctypes.data_as(dp))
    if st != 0:
        raise MMOTError(st, lib.mmot_last_error(None).decode())
    return fin, bin_


def compose_rank_affine(l: int, elems_all, world: int, rank: int):
    """Host reference of the sharded restricted-scan composition (C ABI, no GPU needed).
    elems_all: float64 array [world][2][l * 2**(l-2)].  Returns (fin, bin) arrays of 2**(l-2)."""
    import numpy as np
    lib = load_library()
    a = np.ascontiguousarray(elems_all, dtype=np.float64)
    MO = 1 << (l - 2)
    fin, bin_ = np.zeros(MO), np.zeros(MO)
    dp = ctypes.POINTER(ctypes.c_double)
    st = lib.mmot_compose_rank_affine(int(l), a.ctypes.data_as(dp), int(world), int(rank), fin.ctypes.data_as(dp),
                                      bin_.ctypes.data_as(dp))
    if st != 0:
        raise MMOTError(st, lib.mmot_last_error(None).decode())
    return fin, bin_


class VirtualGroup:
    """In-process group of `world` virtual shards on one device (mmot_vgroup_create): pass
    ``shard=(rank, world, group)`` to Context from one host thread per rank."""

    def __init__(self, world: int):
        self._lib = load_library()
        self.world = int(world)
        g = ctypes.c_void_p()
        st = self._lib.mmot_vgroup_create(self.world, ctypes.byref(g))
        if st != 0:
            raise MMOTError(st, self._lib.mmot_last_error(None).decode())
        self._g = g

    def close(self) -> None:
        if getattr(self, "_g", None):
            self._lib.mmot_vgroup_destroy(self._g)
            self._g = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Context:
    """One MMOT problem shape (l, N, eta, grid) with its device workspace.

    Tensors passed in are torch CUDA tensors (float64, contiguous); the binding only
    forwards their data pointers and the current CUDA stream to the C ABI.
    """

    def __init__(self, l: int, N: int, eta, grid=(0.0, 1.0), dtype: str = "f64",
                 repr: str = "log", check_every: int = 0, chunk: int = 0, stream=None,
                 kernel: str = "auto", batch: Optional[int] = None, shard=None, points=None, shape2d=None):
        """Single instance (eta: float), or a batched context (batch=B, eta: B per-instance
        values) whose array arguments are [B][N] planes (mmot_create_batched).  points: N strictly
        increasing grid coordinates for a non-uniform grid (mmot_create_points / _batched_points).
        shape2d=(N1, N2): a 2-D N1 x N2 mesh (mmot_create_2d, l = 3), N = N1 N2, vectors column-major,
        grid = (x_min, x_max, y_min, y_max)."""
        import torch
        self._lib = load_library()
        if not torch.cuda.is_available():
            raise MMOTError(7, "no CUDA device: the library has no CPU path")
        self.batch = None if batch is None else int(batch)
        self.l, self.N = int(l), int(N)
        self.eta = float(eta) if self.batch is None else [float(e) for e in eta]
        self.shape2d = None if shape2d is None else (int(shape2d[0]), int(shape2d[1]))
        if self.shape2d is not None:
            g4 = tuple(float(v) for v in grid) if len(grid) == 4 else (0.0, 1.0, 0.0, 1.0)
            grid = g4[:2]
        self.grid = (float(grid[0]), float(grid[1]))
        self.repr = repr
        if dtype not in ("f64", "f32"):
            raise MMOTError(1, f"dtype must be 'f64' or 'f32', got {dtype!r}")
        self.dtype = dtype  # f32: float marginals / marginal outputs (fp32 I/O), fp64 scans; u[] stays float64
        self.h = (self.grid[1] - self.grid[0]) / (self.N - 1) if self.N > 1 else 1.0
        self.stream = stream if stream is not None else torch.cuda.current_stream()
        kern = {"auto": 0, "two_walk": 1, "single_walk": 2, "persistent": 3, "stable": 4}[kernel]
        opts = _Opts(int(check_every), 0, LOG if repr == "log" else LINEAR, int(chunk), kern)
        ctx = ctypes.c_void_p()
        self.shard = shard
        if self.shape2d is not None:
            N1, N2 = self.shape2d
            if N1 * N2 != self.N:
                raise MMOTError(2, f"shape2d {self.shape2d} does not hold N = {self.N} points")
            st = self._lib.mmot_create_2d(self.l, N1, N2, float(eta), _Grid2d(*g4), F64 if dtype == "f64" else F32,
                                          ctypes.byref(opts), ctypes.c_void_p(self.stream.cuda_stream),
                                          ctypes.byref(ctx))
            if st != 0:
                raise MMOTError(st, self._lib.mmot_last_error(None).decode())
            self._ctx = ctx
            self.shard = None
            return
        if shard is not None and points is not None:
            raise MMOTError(10, "sharded contexts support uniform grids only")
        if shard is not None:
            rank, world, uid = shard
            self.N_global = self.N
            lo, hi = shard_range(self.N, rank, world)
            self.N = hi - lo
            if isinstance(uid, VirtualGroup):
                st = self._lib.mmot_create_sharded_virtual(self.l, self.N_global, float(eta), _Grid(*self.grid),
                                                           F64 if dtype == "f64" else F32, uid._g, int(rank),
                                                           ctypes.byref(opts), ctypes.c_void_p(self.stream.cuda_stream),
                                                           ctypes.byref(ctx))
                if st != 0:
                    raise MMOTError(st, self._lib.mmot_last_error(None).decode())
                self._ctx = ctx
                return
            idb = ctypes.create_string_buffer(bytes(uid), 128)
            st = self._lib.mmot_create_sharded(self.l, self.N_global, float(eta), _Grid(*self.grid),
                                               F64 if dtype == "f64" else F32, idb, int(rank), int(world),
                                               ctypes.byref(opts), ctypes.c_void_p(self.stream.cuda_stream),
                                               ctypes.byref(ctx))
        elif points is not None:
            xs = [float(v) for v in points]
            if len(xs) != self.N:
                raise MMOTError(2, f"expected {self.N} grid points, got {len(xs)}")
            self.grid = (xs[0], xs[-1])
            self.h = None
            xa = (ctypes.c_double * self.N)(*xs)
            if self.batch is None:
                st = self._lib.mmot_create_points(self.l, self.N, self.eta, xa, F64 if dtype == "f64" else F32,
                                                  ctypes.byref(opts), ctypes.c_void_p(self.stream.cuda_stream),
                                                  ctypes.byref(ctx))
            else:
                etas = (ctypes.c_double * self.batch)(*self.eta)
                st = self._lib.mmot_create_batched_points(self.l, self.N, self.batch, etas, xa,
                                                          F64 if dtype == "f64" else F32, ctypes.byref(opts),
                                                          ctypes.c_void_p(self.stream.cuda_stream), ctypes.byref(ctx))
        elif self.batch is None:
            st = self._lib.mmot_create(self.l, self.N, self.eta, _Grid(*self.grid), F64 if dtype == "f64" else F32,
                                       ctypes.byref(opts), ctypes.c_void_p(self.stream.cuda_stream), ctypes.byref(ctx))
        else:
            if len(self.eta) != self.batch:
                raise MMOTError(2, f"expected {self.batch} eta values, got {len(self.eta)}")
            etas = (ctypes.c_double * self.batch)(*self.eta)
            st = self._lib.mmot_create_batched(self.l, self.N, self.batch, etas, _Grid(*self.grid),
                                               F64 if dtype == "f64" else F32, ctypes.byref(opts),
                                               ctypes.c_void_p(self.stream.cuda_stream), ctypes.byref(ctx))
        if st != 0:
            raise MMOTError(st, self._lib.mmot_last_error(None).decode())
        self._ctx = ctx

    # -- helpers ------------------------------------------------------------------------
    def _check(self, st: int):
        if st != 0:
            raise MMOTError(st, self._lib.mmot_last_error(self._ctx).decode())

    def _ptrs(self, ts) -> ctypes.Array:
        if len(ts) != self.l:
            raise MMOTError(2, f"expected {self.l} vectors, got {len(ts)}")
        n = self.N * (self.batch or 1)
        for t in ts:
            if not t.is_cuda or not t.is_contiguous() or t.numel() != n:
                raise MMOTError(2, f"vectors must be contiguous CUDA tensors of {n} elements")
        return _ptr_array([t.data_ptr() for t in ts])

    @property
    def info(self) -> dict:
        """Launch plan: chain length P, number of chains, kernel family ("two_walk"/"single_walk")."""
        P, n, k = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int()
        self._check(self._lib.mmot_info(self._ctx, ctypes.byref(P), ctypes.byref(n), ctypes.byref(k)))
        return dict(chain_len=P.value, nchains=n.value,
                    kernel={1: "two_walk", 2: "single_walk", 3: "persistent", 4: "stable", 5: "grid2d",
                            6: "lanes"}[k.value])

    @property
    def launches(self) -> int:
        return int(self._lib.mmot_launch_count(self._ctx))

    @property
    def stable_fallbacks(self) -> int:
        """Calls redone on the stabilised (log-domain) family after a product left the fp64 range."""
        return int(self._lib.mmot_stable_fallback_count(self._ctx))

    @property
    def allres_checks(self) -> int:
        """Residual checks evaluated by the single all-marginals pass (NEXT-1)."""
        return int(self._lib.mmot_allres_checks(self._ctx))

    @property
    def graph_solves(self) -> int:
        """Solves whose sweep loop ran as one device-resident CUDA graph launch."""
        return int(self._lib.mmot_graph_solves(self._ctx))

    @property
    def pair_solves(self) -> int:
        """Batched solves that ran on the pair family (two threads per instance, no chain operators)."""
        return int(self._lib.mmot_pair_solves(self._ctx))

    @property
    def pair_f32_solves(self) -> int:
        """Pair-family solves that computed in fp32 arithmetic (MMOT_F32 contexts; slab exponents)."""
        return int(self._lib.mmot_pair_f32_solves(self._ctx))

    @property
    def pair_redo(self) -> int:
        """Instances of fp32 pair solves redone in fp64 after their states left the fp32 range."""
        return int(self._lib.mmot_pair_redo_count(self._ctx))

    @property
    def cta_solves(self) -> int:
        """Batched / small-instance solves that ran on the CTA family (a thread block per instance)."""
        return int(self._lib.mmot_cta_solves(self._ctx))

    @property
    def fallbacks(self) -> int:
        """Calls redone on the two-walk family after the single-walk precision guard tripped."""
        return int(self._lib.mmot_fallback_count(self._ctx))

    # -- ABI calls ------------------------------------------------------------------------
    def init_uniform(self, u) -> None:
        self._check(self._lib.mmot_init_uniform(self._ctx, self._ptrs(u)))

    def marginal(self, k: int, u, out=None):
        import torch
        if out is None:
            shape = (self.N,) if self.batch is None else (self.batch, self.N)
            out = torch.empty(shape, dtype=torch.float32 if self.dtype == "f32" else torch.float64, device=u[0].device)
        self._check(self._lib.mmot_marginal(self._ctx, int(k), self._ptrs(u), ctypes.c_void_p(out.data_ptr())))
        return out

    def sinkhorn(self, marginals, iters: int, tol: float, u) -> dict:
        import torch
        want = torch.float32 if self.dtype == "f32" else torch.float64
        if any(m.dtype != want for m in marginals) or any(x.dtype != torch.float64 for x in u):
            raise MMOTError(2, f"marginals must be {want} and u float64 for a {self.dtype} context")
        rep = _Report()
        st = self._lib.mmot_sinkhorn(self._ctx, self._ptrs(marginals), int(iters), float(tol), self._ptrs(u),
                                     ctypes.byref(rep))
        out = dict(iters_done=rep.iters_done, residual=rep.residual, converged=bool(rep.converged),
                   status=rep.status, fail_iter=rep.fail_iter)
        if st != 0:
            err = MMOTError(st, self._lib.mmot_last_error(self._ctx).decode())
            err.report = out
            raise err
        return out

    def sinkhorn_host(self, marginals_host, iters: int, tol: float, u_host) -> dict:
        """Host (pinned torch CPU or numpy) buffers; copies happen inside the call."""
        def hp(a):
            return a.data_ptr() if hasattr(a, "data_ptr") else a.ctypes.data
        rep = _Report()
        st = self._lib.mmot_sinkhorn_host(self._ctx, _ptr_array([hp(a) for a in marginals_host]), int(iters),
                                          float(tol), _ptr_array([hp(a) for a in u_host]), ctypes.byref(rep))
        self._check(st)
        return dict(iters_done=rep.iters_done, residual=rep.residual, converged=bool(rep.converged),
                    status=rep.status, fail_iter=rep.fail_iter)

    def cost(self, u):
        """W (float), or for a batched context a list of the B per-instance costs."""
        if self.batch is not None:
            Wb = (ctypes.c_double * self.batch)()
            self._check(self._lib.mmot_cost(self._ctx, self._ptrs(u), Wb))
            return list(Wb)
        W = ctypes.c_double()
        self._check(self._lib.mmot_cost(self._ctx, self._ptrs(u), ctypes.byref(W)))
        return W.value

    def cost_staged(self):
        """W of the scalings the last sinkhorn_host left on the device (mmot_cost_staged)."""
        Wb = (ctypes.c_double * (self.batch or 1))()
        self._check(self._lib.mmot_cost_staged(self._ctx, Wb))
        return list(Wb) if self.batch is not None else Wb[0]

    def profile(self, enable: bool = True) -> None:
        self._check(self._lib.mmot_profile_enable(self._ctx, 1 if enable else 0))

    def profile_read(self) -> dict:
        """Device ms per product phase (ops, scan, apply, total) and per mode since the last read."""
        ms = (ctypes.c_double * 4)()
        msm = (ctypes.c_double * 4)()
        nm = (ctypes.c_int64 * 4)()
        self._check(self._lib.mmot_profile_read(self._ctx, ms, msm, nm))
        modes = ["marginal", "update", "residual", "cost"]
        return dict(phase_ms=dict(ops=ms[0], scan=ms[1], apply=ms[2], total=ms[3]),
                    mode_ms={m: msm[i] for i, m in enumerate(modes)},
                    mode_n={m: int(nm[i]) for i, m in enumerate(modes)})

    def close(self) -> None:
        if getattr(self, "_ctx", None):
            self._lib.mmot_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()
