"""Thin ctypes binding of libfftpde.so (include/fftpde.h).

Argument marshalling only: every step of the path runs in the library's sm_100a
kernels.  PyTorch provides device memory (the workspace and outputs are torch
tensors) and the stream (``torch.cuda.current_stream()``).  There is no CPU
fallback: if the library or a CUDA device is missing, the calls raise.

Tensors are ``[ny, nx]`` or ``[B, ny, nx]`` complex128 / complex64, C-contiguous,
x fastest.  Inputs may live on the host (CPU tensors): they
are staged through pinned memory to the plan's device and the result is copied
back, all on the current stream (this is what bench.py's ``e2e`` times).
"""
from __future__ import annotations

import ctypes
import os

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libfftpde.so")

KERNEL_CLASSES = {0: "row_pass", 1: "col_pass", 2: "wave_col_pass", 3: "small_solve", 4: "pointwise",
                  5: "aa_pass"}

# fftpde_status
OK, ERR_INVALID_ARG, ERR_EMPTY, ERR_NOT_POW2_X, ERR_NOT_POW2_Y, ERR_UNSUPPORTED, ERR_WORKSPACE, \
    ERR_CUDA, ERR_NCCL, ERR_NOT_POW2_Z = range(10)
C64, C128 = 0, 1

EXPORTS = [
    "fftpde_plan_2d", "fftpde_workspace_size", "fftpde_set_workspace", "fftpde_set_stream",
    "fftpde_destroy", "fftpde_status_string", "fftpde_launch_count",
    "fftpde_set_profiling", "fftpde_read_profile", "fftpde_nccl_unique_id", "fftpde_plan_2d_sharded",
    "fftpde_plan_3d_sharded", "fftpde_plan_3d_pencil",
    "fftpde_forward", "fftpde_inverse", "fftpde_poisson", "fftpde_diffuse", "fftpde_wave_step",
    "fftpde_forward_batched", "fftpde_inverse_batched", "fftpde_poisson_batched",
    "fftpde_diffuse_batched", "fftpde_wave_step_batched",
    "fftpde_rows", "fftpde_cols_slab", "fftpde_pack_blocks",
    "fftpde_wave_rk4_scratch_size", "fftpde_wave_rk4",
    "fftpde_apply", "fftpde_diffuse_source_scratch_size", "fftpde_diffuse_source",
    "fftpde_plan_3d", "fftpde_plan_2d_r2c", "fftpde_peer_transpose", "fftpde_rows_to_peers",
    "fftpde_cols_to_peers", "fftpde_fs_part_aa", "fftpde_fs_part_b", "fftpde_fs_part_perm",
]
KOP = {"laplacian": 0, "dx": 1, "dy": 2}
OP_POISSON, OP_DIFFUSE, OP_DIFFUSE_Y = 2, 3, 5
ROWS_FWD, ROWS_DIFFUSE = 0, 3


class FFTPDEError(RuntimeError):
    def __init__(self, status: int, what: str):
        self.status = status
        super().__init__(f"{what}: {status_string(status)} (status {status})")


_lib = None


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libfftpde.so (built in-tree by __graft_entry__.build()); raises if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"libfftpde.so not found at {path}: run __graft_entry__.build() "
                           "(there is no CPU fallback)")
    L = ctypes.CDLL(path)
    p, i64, dbl, u = ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_int
    st = ctypes.c_int
    sig = {
        "fftpde_plan_2d": (st, [ctypes.POINTER(p), i64, i64, i64, u, dbl, dbl, u]),
        "fftpde_workspace_size": (ctypes.c_size_t, [p]),
        "fftpde_set_workspace": (st, [p, p, ctypes.c_size_t]),
        "fftpde_set_stream": (st, [p, p]),
        "fftpde_destroy": (st, [p]),
        "fftpde_status_string": (ctypes.c_char_p, [st]),
        "fftpde_launch_count": (i64, [p]),
        "fftpde_set_profiling": (st, [p, u]),
        "fftpde_read_profile": (st, [p, u, ctypes.POINTER(dbl), ctypes.POINTER(i64)]),
        "fftpde_forward": (st, [p, p, p]),
        "fftpde_inverse": (st, [p, p, p]),
        "fftpde_poisson": (st, [p, p, p]),
        "fftpde_diffuse": (st, [p, p, p, dbl, dbl, i64]),
        "fftpde_wave_step": (st, [p, p, p, dbl, dbl, i64]),
        "fftpde_forward_batched": (st, [p, p, p, i64, i64]),
        "fftpde_inverse_batched": (st, [p, p, p, i64, i64]),
        "fftpde_poisson_batched": (st, [p, p, p, i64, i64]),
        "fftpde_diffuse_batched": (st, [p, p, p, i64, i64, dbl, dbl, i64]),
        "fftpde_wave_step_batched": (st, [p, p, p, i64, i64, dbl, dbl, i64]),
        "fftpde_rows": (st, [p, p, p, i64, u]),
        "fftpde_cols_slab": (st, [p, p, p, i64, i64, u, dbl, dbl]),
        "fftpde_pack_blocks": (st, [p, p, p, i64, i64, i64, u]),
        "fftpde_wave_rk4_scratch_size": (ctypes.c_size_t, [p]),
        "fftpde_apply": (st, [p, p, p, u]),
        "fftpde_plan_3d": (st, [ctypes.POINTER(p), i64, i64, i64, u, dbl, dbl, dbl, u]),
        "fftpde_plan_2d_r2c": (st, [ctypes.POINTER(p), i64, i64, i64, u, dbl, dbl, u]),
        "fftpde_nccl_unique_id": (st, [p]),
        "fftpde_plan_2d_sharded": (st, [ctypes.POINTER(p), i64, i64, u, dbl, dbl, u, p, u, u]),
        "fftpde_plan_3d_sharded": (st, [ctypes.POINTER(p), i64, i64, i64, u, dbl, dbl, dbl, u, p, u, u]),
        "fftpde_plan_3d_pencil": (st, [ctypes.POINTER(p), i64, i64, i64, u, dbl, dbl, dbl, u, p, u, u, u]),
        "fftpde_peer_transpose": (st, [p, p, ctypes.POINTER(p), u, u, i64, i64, u]),
        "fftpde_rows_to_peers": (st, [p, p, ctypes.POINTER(p), u, u, i64, u, dbl, dbl]),
        "fftpde_cols_to_peers": (st, [p, p, ctypes.POINTER(p), u, u, i64, u, dbl, dbl]),
        "fftpde_fs_part_aa": (st, [p, u, u, u, u, p, p, p]),
        "fftpde_fs_part_b": (st, [p, u, u, u, p, dbl, dbl, ctypes.POINTER(p), u]),
        "fftpde_fs_part_perm": (st, [p, u, p, p, u]),
        "fftpde_diffuse_source_scratch_size": (ctypes.c_size_t, [p]),
        "fftpde_diffuse_source": (st, [p, p, p, p, dbl, dbl, i64, p, ctypes.c_size_t]),
        "fftpde_wave_rk4": (st, [p, p, p, dbl, dbl, dbl, dbl, dbl, dbl, dbl, dbl, dbl, dbl, i64, p, p,
                                 ctypes.c_size_t]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def status_string(status: int) -> str:
    return load_library().fftpde_status_string(status).decode()


def _check(status: int, what: str):
    if status != OK:
        raise FFTPDEError(status, what)


_DT = {torch.complex128: C128, torch.complex64: C64}


class Plan:
    """A 2D FFT-PDE plan for ``batch`` grids of ``ny x nx`` on [0,Lx) x [0,Ly).

    Mirrors fftpde_plan_2d + workspace (a torch uint8 tensor) + stream."""

    def __init__(self, nx: int, ny: int, batch: int = 1, dtype=torch.complex128,
                 Lx: float = 1.0, Ly: float = 1.0, device=None):
        if dtype not in _DT:
            raise TypeError("dtype must be torch.complex128 or torch.complex64")
        if not torch.cuda.is_available():
            raise RuntimeError("fftpde needs a CUDA device (no CPU fallback)")
        self.lib = load_library()
        self.device = torch.device(device if device is not None else "cuda", )
        if self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        self.nx, self.ny, self.batch, self.dtype = int(nx), int(ny), int(batch), dtype
        self.Lx, self.Ly = float(Lx), float(Ly)
        h = ctypes.c_void_p()
        _check(self.lib.fftpde_plan_2d(ctypes.byref(h), self.nx, self.ny, self.batch, _DT[dtype],
                                       self.Lx, self.Ly, self.device.index), "fftpde_plan_2d")
        self._h = h
        nbytes = self.lib.fftpde_workspace_size(h)
        self.workspace = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=self.device)
        self._bind_stream()
        _check(self.lib.fftpde_set_workspace(h, self.workspace.data_ptr(), self.workspace.numel()),
               "fftpde_set_workspace")

    # -- plumbing -----------------------------------------------------------------
    def _bind_stream(self):
        # the raw cudaStream_t of torch's current stream; the library is told only
        # when it changes (a per-call set_stream would cost host time per solve)
        s = torch._C._cuda_getCurrentRawStream(self.device.index)
        if s != getattr(self, "_stream", None):
            _check(self.lib.fftpde_set_stream(self._h, s), "fftpde_set_stream")
            self._stream = s

    def close(self):
        if getattr(self, "_h", None):
            self.lib.fftpde_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def launches(self) -> int:
        return int(self.lib.fftpde_launch_count(self._h))

    def set_profiling(self, enable: bool):
        _check(self.lib.fftpde_set_profiling(self._h, int(bool(enable))), "fftpde_set_profiling")

    def read_profile(self) -> dict:
        """{kernel class: (total device ms, launches)} since the last read."""
        out = {}
        for cls, name in KERNEL_CLASSES.items():
            ms, n = ctypes.c_double(), ctypes.c_int64()
            _check(self.lib.fftpde_read_profile(self._h, cls, ctypes.byref(ms), ctypes.byref(n)),
                   "fftpde_read_profile")
            if n.value:
                out[name] = (ms.value, n.value)
        return out

    def _grid(self, x: torch.Tensor, name: str):
        if x.dtype != self.dtype:
            raise TypeError(f"{name}: dtype {x.dtype} does not match the plan's {self.dtype}")
        if x.dim() == 2:
            B = 1
        elif x.dim() == 3:
            B = x.shape[0]
        else:
            raise ValueError(f"{name}: expected [ny, nx] or [B, ny, nx]")
        if tuple(x.shape[-2:]) != (self.ny, self.nx):
            raise ValueError(f"{name}: shape {tuple(x.shape)} does not match plan ({self.ny}, {self.nx})")
        if B > self.batch:
            raise ValueError(f"{name}: batch {B} exceeds the plan's {self.batch}")
        return B

    def _to_dev(self, x: torch.Tensor):
        """(device tensor, was_host).  Host tensors go through pinned memory."""
        if x.device.type == "cpu":
            src = x.contiguous()
            if not src.is_pinned():
                src = src.pin_memory()
            return src.to(self.device, non_blocking=True), True
        if x.device != self.device:
            raise ValueError(f"tensor on {x.device}, plan on {self.device}")
        return x.contiguous(), False

    def _finish(self, out_dev: torch.Tensor, host: bool, host_out=None):
        """Device result, or (host inputs) its copy in pinned host memory
        (``host_out`` if given, a pinned tensor of the right shape)."""
        if host:
            out = host_out if host_out is not None else torch.empty(out_dev.shape, dtype=out_dev.dtype,
                                                                    pin_memory=True)
            out.copy_(out_dev, non_blocking=True)
            torch.cuda.current_stream(self.device).synchronize()
            return out
        return out_dev

    def _out(self, like: torch.Tensor, out):
        if out is None:
            return torch.empty_like(like)
        if out.shape != like.shape or out.dtype != like.dtype or out.device != like.device \
                or not out.is_contiguous():
            raise ValueError("out: must be a contiguous tensor like the input on the plan's device")
        return out

    # -- transforms and solvers -----------------------------------------------------
    def forward(self, x: torch.Tensor, out=None) -> torch.Tensor:
        """DFT2 with the paper's + sign, unnormalised."""
        B = self._grid(x, "x")
        xd, host = self._to_dev(x)
        o = self._out(xd, None if host else out)
        self._bind_stream()
        _check(self.lib.fftpde_forward_batched(self._h, xd.data_ptr(), o.data_ptr(), B,
                                               self.nx * self.ny), "fftpde_forward")
        return self._finish(o, host, out if host else None)

    def inverse(self, X: torch.Tensor, out=None) -> torch.Tensor:
        """iDFT2: conjugate kernel, times 1/(nx ny)."""
        B = self._grid(X, "X")
        xd, host = self._to_dev(X)
        o = self._out(xd, None if host else out)
        self._bind_stream()
        _check(self.lib.fftpde_inverse_batched(self._h, xd.data_ptr(), o.data_ptr(), B,
                                               self.nx * self.ny), "fftpde_inverse")
        return self._finish(o, host, out if host else None)

    def poisson(self, rho: torch.Tensor, out=None) -> torch.Tensor:
        """u with nabla^2 u = rho - mean(rho), zero mean (eq:SolutionPoisson)."""
        B = self._grid(rho, "rho")
        rd, host = self._to_dev(rho)
        o = self._out(rd, None if host else out)
        self._bind_stream()
        _check(self.lib.fftpde_poisson_batched(self._h, rd.data_ptr(), o.data_ptr(), B,
                                               self.nx * self.ny), "fftpde_poisson")
        return self._finish(o, host, out if host else None)

    def diffuse(self, u0: torch.Tensor, D: float, dt: float, nsteps: int, out=None) -> torch.Tensor:
        """nsteps exact diffusion steps exp(-D|k|^2 dt) (ec:solCalorFourier)."""
        B = self._grid(u0, "u0")
        ud, host = self._to_dev(u0)
        o = self._out(ud, None if host else out)
        self._bind_stream()
        _check(self.lib.fftpde_diffuse_batched(self._h, ud.data_ptr(), o.data_ptr(), B,
                                               self.nx * self.ny, float(D), float(dt), int(nsteps)),
               "fftpde_diffuse")
        return self._finish(o, host, out if host else None)

    def wave_step(self, u: torch.Tensor, ut: torch.Tensor, c: float, dt: float, nsteps: int):
        """nsteps exact wave steps on (u, ut) (eq:OmegaZero/NonZero).

        Device tensors are updated in place and returned; host tensors are copied."""
        B = self._grid(u, "u")
        if self._grid(ut, "ut") != B:
            raise ValueError("u and ut batch differ")
        ud, host = self._to_dev(u)
        vd, _ = self._to_dev(ut)
        if not host and (ud.data_ptr() != u.data_ptr() or vd.data_ptr() != ut.data_ptr()):
            raise ValueError("wave_step updates in place: pass contiguous device tensors")
        self._bind_stream()
        _check(self.lib.fftpde_wave_step_batched(self._h, ud.data_ptr(), vd.data_ptr(), B,
                                                 self.nx * self.ny, float(c), float(dt), int(nsteps)),
               "fftpde_wave_step")
        if host:
            return self._finish(ud, True), self._finish(vd, True)
        return ud, vd

    def apply(self, x: torch.Tensor, op: str, out=None) -> torch.Tensor:
        """iDFT2(m .* DFT2(x)): m = -|k|^2 ("laplacian"), -i kx ("dx"), -i ky ("dy")
        (F{du/dx} = -i w F{u}) over the plan's whole batch."""
        if self._grid(x, "x") != self.batch:
            raise ValueError("apply acts on the plan's whole batch")
        xd, host = self._to_dev(x)
        o = self._out(xd, None if host else out)
        self._bind_stream()
        _check(self.lib.fftpde_apply(self._h, xd.data_ptr(), o.data_ptr(), KOP[op]), "fftpde_apply")
        return self._finish(o, host, out if host else None)

    def diffuse_source(self, u0: torch.Tensor, s: torch.Tensor, D: float, dt: float, nsteps: int,
                       out=None) -> torch.Tensor:
        """nsteps exact steps of u_t = D nabla^2 u + s, static s."""
        if self._grid(u0, "u0") != self.batch or self._grid(s, "s") != self.batch:
            raise ValueError("diffuse_source acts on the plan's whole batch")
        ud, host = self._to_dev(u0)
        sd, _ = self._to_dev(s)
        o = self._out(ud, None if host else out)
        nbytes = int(self.lib.fftpde_diffuse_source_scratch_size(self._h))
        if getattr(self, "_ds_scratch", None) is None or self._ds_scratch.numel() < nbytes:
            self._ds_scratch = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        self._bind_stream()
        _check(self.lib.fftpde_diffuse_source(self._h, ud.data_ptr(), sd.data_ptr(), o.data_ptr(), float(D),
                                              float(dt), int(nsteps), self._ds_scratch.data_ptr(),
                                              self._ds_scratch.numel()), "fftpde_diffuse_source")
        return self._finish(o, host, out if host else None)

    def wave_rk4(self, u: torch.Tensor, ut: torch.Tensor, dt: float, nsteps: int, c: float = 1.0,
                 t0: float = 0.0, xmin: float = 0.0, ymin: float = 0.0, A: float = 1.0,
                 sigma: float = 0.1, Omega: float = 5.0, gamma: float = 10.0, rs: float = 0.5):
        """nsteps RK4 steps of u_tt = c^2 nabla^2 u + s with the orbiting Gaussian
        source on the plan's grid x_j = xmin + j Lx/nx.

        (u, ut) are device tensors updated in place; returns the grid means of u at
        t0 + n dt, n = 0..nsteps (a device tensor of the plan's dtype)."""
        if self._grid(u, "u") != 1 or self._grid(ut, "ut") != 1 or u.dim() != 2:
            raise ValueError("wave_rk4: expects [ny, nx] fields (batch 1)")
        for x, name in ((u, "u"), (ut, "ut")):
            if x.device != self.device or not x.is_contiguous():
                raise ValueError(f"wave_rk4 updates in place: {name} must be a contiguous device tensor")
        nbytes = int(self.lib.fftpde_wave_rk4_scratch_size(self._h))
        if getattr(self, "_rk4_scratch", None) is None or self._rk4_scratch.numel() < nbytes:
            self._rk4_scratch = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        means = torch.empty(int(nsteps) + 1, dtype=self.dtype, device=self.device)
        self._bind_stream()
        _check(self.lib.fftpde_wave_rk4(self._h, u.data_ptr(), ut.data_ptr(), float(c), float(xmin),
                                        float(ymin), float(A), float(sigma), float(Omega), float(gamma),
                                        float(rs), float(t0), float(dt), int(nsteps), means.data_ptr(),
                                        self._rk4_scratch.data_ptr(), self._rk4_scratch.numel()),
               "fftpde_wave_rk4")
        return means

    # -- slab (sharded) building blocks ------------------------------------------------
    def _dense(self, name: str, *ts: torch.Tensor, numel: int = 0):
        """The slab kernels take raw pointers to dense buffers: every tensor must be a
        contiguous tensor of the plan's dtype on the plan's device holding at least
        `numel` elements (an undersized buffer would be written out of bounds)."""
        for t in ts:
            if not isinstance(t, torch.Tensor) or t.device != self.device or t.dtype != self.dtype \
                    or not t.is_contiguous():
                raise ValueError(f"{name}: expected contiguous {self.dtype} tensors on {self.device}")
            if t.numel() < numel:
                raise ValueError(f"{name}: buffer of {t.numel()} elements, the call touches {numel}")

    def rows(self, x: torch.Tensor, out: torch.Tensor, inverse: bool = False):
        """Transforms along x of the rows of a [nrows, nx] device slab (any nrows)."""
        if x.dim() != 2 or x.shape[1] != self.nx or out.shape != x.shape or x.dtype != self.dtype:
            raise ValueError("rows: expected matching [nrows, nx] tensors of the plan's dtype")
        self._dense("rows", x, out)
        self._bind_stream()
        _check(self.lib.fftpde_rows(self._h, x.data_ptr(), out.data_ptr(), x.shape[0], int(inverse)),
               "fftpde_rows")
        return out

    def cols_slab(self, x: torch.Tensor, out: torch.Tensor, col0: int, op: int, D: float = 0.0,
                  dt: float = 0.0):
        """Column pass (forward, operator at the global wavenumbers, inverse) of a
        [ny, ncols] column slab holding global columns col0 .. col0+ncols-1."""
        if x.dim() != 2 or x.shape[0] != self.ny or out.shape != x.shape or x.dtype != self.dtype:
            raise ValueError("cols_slab: expected matching [ny, ncols] tensors of the plan's dtype")
        self._dense("cols_slab", x, out)
        self._bind_stream()
        _check(self.lib.fftpde_cols_slab(self._h, x.data_ptr(), out.data_ptr(), int(col0), x.shape[1],
                                         int(op), float(D), float(dt)), "fftpde_cols_slab")
        return out

    def peer_transpose(self, src: torch.Tensor, peers, rank: int, R: int, bw: int, direction: int):
        """Slab exchange by direct stores into the peers' buffers (fftpde_peer_transpose);
        peers: device pointers (ints) of every rank's destination buffer."""
        self._dense("peer_transpose", src, numel=int(R) * self.nx)
        if len(peers) < 1 or int(bw) * len(peers) != self.nx:
            raise ValueError("peer_transpose: expected one destination per rank and bw * P == nx")
        arr = (ctypes.c_void_p * len(peers))(*[int(x) for x in peers])
        self._bind_stream()
        _check(self.lib.fftpde_peer_transpose(self._h, src.data_ptr(), arr, len(peers), int(rank), int(R), int(bw),
                                              int(direction)), "fftpde_peer_transpose")

    def rows_to_peers(self, x: torch.Tensor, peers, rank: int, R: int, op: int = 0, D: float = 0.0,
                      dt: float = 0.0):
        """Row pass of this rank's [R, nx] slab with its output stored straight into
        the peers' [ny, nx/P] column slabs (fftpde_rows_to_peers: the exchange fused
        into the row pass); op 0 = forward transform, 3 = x diffusion (R26)."""
        if x.dim() != 2 or tuple(x.shape) != (R, self.nx) or x.dtype != self.dtype or not x.is_contiguous():
            raise ValueError("rows_to_peers: expected a contiguous [R, nx] slab of the plan's dtype")
        arr = (ctypes.c_void_p * len(peers))(*[int(q) for q in peers])
        self._bind_stream()
        _check(self.lib.fftpde_rows_to_peers(self._h, x.data_ptr(), arr, len(peers), int(rank), int(R), int(op),
                                             float(D), float(dt)), "fftpde_rows_to_peers")

    def cols_to_peers(self, cs: torch.Tensor, peers, rank: int, R: int, op: int, D: float = 0.0, dt: float = 0.0):
        """Column pass of this rank's [ny, nx/P] column slab with its output stored
        straight into the owners' [R, nx] row slabs (fftpde_cols_to_peers: the return
        exchange fused into the column pass); the slab is used as scratch."""
        if cs.dim() != 2 or cs.shape[0] != self.ny or cs.dtype != self.dtype or not cs.is_contiguous():
            raise ValueError("cols_to_peers: expected a contiguous [ny, nx/P] slab of the plan's dtype")
        arr = (ctypes.c_void_p * len(peers))(*[int(q) for q in peers])
        self._bind_stream()
        _check(self.lib.fftpde_cols_to_peers(self._h, cs.data_ptr(), arr, len(peers), int(rank), int(R), int(op),
                                             float(D), float(dt)), "fftpde_cols_to_peers")

    # ---- the distributed four-step pieces (R28; 32768^2 complex128 plans) ----
    def fs_part_aa(self, op: int, P: int, rank: int, xmode: int, x: torch.Tensor, out: torch.Tensor,
                   phys: torch.Tensor = None):
        """AA (op 0) / AA^-1 (1) / MID (2) on this rank's part [P][32][M][32][M] (fftpde_fs_part_aa)."""
        n = self.nx * self.ny // int(P)
        self._dense("fs_part_aa", x, out, *([phys] if phys is not None else []), numel=n)
        self._bind_stream()
        _check(self.lib.fftpde_fs_part_aa(self._h, int(op), int(P), int(rank), int(xmode), x.data_ptr(),
                                          out.data_ptr(), phys.data_ptr() if phys is not None else None),
               "fftpde_fs_part_aa")

    def fs_part_b(self, xmode: int, P: int, rank: int, f: torch.Tensor, D: float, dt: float, peers=None):
        """The 1024-point diffusion pass of the part's local axis, in place or (peers: every
        rank's other-part pointer) stored straight into the peers' other part (fftpde_fs_part_b)."""
        self._dense("fs_part_b", f, numel=self.nx * self.ny // int(P))
        arr = (ctypes.c_void_p * len(peers))(*[int(q) for q in peers]) if peers is not None else None
        self._bind_stream()
        _check(self.lib.fftpde_fs_part_b(self._h, int(xmode), int(P), int(rank), f.data_ptr(), float(D), float(dt),
                                         arr, len(peers) if peers is not None else 0), "fftpde_fs_part_b")

    def fs_part_perm(self, P: int, x: torch.Tensor, out: torch.Tensor, direction: int):
        """Row slab <-> [P][P][32/P][M][32][M] (fftpde_fs_part_perm)."""
        self._dense("fs_part_perm", x, out, numel=self.nx * self.ny // int(P))
        self._bind_stream()
        _check(self.lib.fftpde_fs_part_perm(self._h, int(P), x.data_ptr(), out.data_ptr(), int(direction)),
               "fftpde_fs_part_perm")

    def peer_blocks(self, src: torch.Tensor, peers, rank: int):
        """All-to-all of equal blocks by peer stores: block q of src -> peers[q] at block `rank`
        (fftpde_peer_transpose with one row)."""
        P = len(peers)
        self._dense("peer_blocks", src)
        if src.numel() % P or (src.numel() // P * src.element_size()) % 16:
            raise ValueError("peer_blocks: src must split into P blocks of whole 16-byte vectors")
        arr = (ctypes.c_void_p * P)(*[int(x) for x in peers])
        self._bind_stream()
        _check(self.lib.fftpde_peer_transpose(self._h, src.data_ptr(), arr, P, int(rank), 1, src.numel() // P, 0),
               "fftpde_peer_transpose")

    def pack_blocks(self, x: torch.Tensor, out: torch.Tensor, nrows: int, nblocks: int, bw: int,
                    direction: int):
        """[nrows][nblocks][bw] <-> [nblocks][nrows][bw] (direction 0 / 1)."""
        self._dense("pack_blocks", x, out, numel=int(nrows) * int(nblocks) * int(bw))
        self._bind_stream()
        _check(self.lib.fftpde_pack_blocks(self._h, x.data_ptr(), out.data_ptr(), int(nrows), int(nblocks),
                                           int(bw), int(direction)), "fftpde_pack_blocks")
        return out


SHARDED_LOOPBACK = -1


def broadcast_unique_id(draw, group=None) -> bytes:
    """The 128-byte NCCL unique id for a sharded plan: ``draw()`` on rank 0 of
    ``group`` (fftpde_nccl_unique_id), broadcast to every rank over the torch
    process group (any backend)."""
    import torch.distributed as dist
    rank = dist.get_rank(group)
    box = [draw() if rank == 0 else None]
    src = dist.get_global_rank(group, 0) if group is not None else 0
    dist.broadcast_object_list(box, src=src, group=group)
    if not isinstance(box[0], (bytes, bytearray)) or len(box[0]) != 128:
        raise RuntimeError("bad NCCL unique id broadcast")
    return bytes(box[0])


class _Sharded(Plan):
    """Common part of ShardedPlan / ShardedPlan3D: communicator set-up and the
    collective whole-plan calls.  ``loopback=P`` builds the single-process
    emulation of P ranks on this device (FFTPDE_SHARDED_LOOPBACK): buffers hold
    the P slabs back to back."""

    def _setup(self, dtype, device, group, loopback, make):
        if dtype not in _DT:
            raise TypeError("dtype must be torch.complex128 or torch.complex64")
        if not torch.cuda.is_available():
            raise RuntimeError("fftpde needs a CUDA device (no CPU fallback)")
        import torch.distributed as dist
        self.lib = load_library()
        self.dtype, self.batch = dtype, 1
        self.device = torch.device(device if device is not None else "cuda")
        if self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        h = ctypes.c_void_p()
        if loopback:
            self.rank, self.P, self.loopback = 0, int(loopback), True
            _check(make(h, None, SHARDED_LOOPBACK, self.P), "sharded plan (loopback)")
        else:
            self.loopback = False
            if dist.is_available() and dist.is_initialized():
                self.rank, self.P = dist.get_rank(group), dist.get_world_size(group)
            else:
                self.rank, self.P = 0, 1

            def draw():
                buf = ctypes.create_string_buffer(128)
                _check(self.lib.fftpde_nccl_unique_id(buf), "fftpde_nccl_unique_id")
                return buf.raw

            uid = draw() if self.P == 1 else broadcast_unique_id(draw, group)
            _check(make(h, ctypes.create_string_buffer(uid, 128), self.rank, self.P), "sharded plan")
        self._h = h
        nbytes = self.lib.fftpde_workspace_size(h)
        self.workspace = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=self.device)
        self._bind_stream()
        _check(self.lib.fftpde_set_workspace(h, self.workspace.data_ptr(), self.workspace.numel()),
               "fftpde_set_workspace")

    def _lb(self, shape):
        return ((self.P,) + shape) if self.loopback else shape

    def _slab(self, x, shape, name):
        if x.dtype != self.dtype or tuple(x.shape) != shape:
            raise ValueError(f"{name}: expected {self.dtype} {shape}, got {x.dtype} {tuple(x.shape)}")
        if x.device != self.device or not x.is_contiguous():
            raise ValueError(f"{name}: expected a contiguous tensor on {self.device}")

    def _run(self, fn, x, xs, os_, out, *args):
        self._slab(x, xs, "input")
        o = torch.empty(os_, dtype=self.dtype, device=self.device) if out is None else out
        self._slab(o, os_, "out")
        self._bind_stream()
        _check(fn(self._h, x.data_ptr(), o.data_ptr(), *args), fn.__name__)
        return o

    def forward(self, x, out=None):
        """Physical slab -> this rank's spectral slab (see the class docstring)."""
        return self._run(self.lib.fftpde_forward, x, self.phys_shape, self.spec_shape, out)

    def inverse(self, X, out=None):
        return self._run(self.lib.fftpde_inverse, X, self.spec_shape, self.phys_shape, out)

    def poisson(self, rho, out=None):
        return self._run(self.lib.fftpde_poisson, rho, self.phys_shape, self.phys_shape, out)

    def diffuse(self, u0, D: float, dt: float, nsteps: int, out=None):
        return self._run(self.lib.fftpde_diffuse, u0, self.phys_shape, self.phys_shape, out,
                         float(D), float(dt), int(nsteps))


class ShardedPlan(_Sharded):
    """The slab decomposition of one ny x nx grid over the ranks of ``group``
    (fftpde_plan_2d_sharded): NCCL runs inside the library on a
    communicator of its own, created from a unique id that rank 0 draws and this
    binding broadcasts over ``group``.  Rank r holds rows [r R, (r+1) R), R = ny/P
    (``phys_shape`` [R, nx]); its spectrum slab is columns [r BW, (r+1) BW),
    BW = nx/P (``spec_shape`` [ny, BW]).  Every call is collective.  Without an
    initialised process group it is a P = 1 plan (NCCL send/recv to itself);
    ``loopback=P`` emulates P ranks in this process ([ny, nx] in, [P, ny, BW] spectra)."""

    def __init__(self, nx: int, ny: int, dtype=torch.complex128, Lx: float = 1.0, Ly: float = 1.0,
                 device=None, group=None, loopback: int = 0):
        self.nx, self.ny, self.Lx, self.Ly = int(nx), int(ny), float(Lx), float(Ly)
        self._setup(dtype, device, group, loopback,
                    lambda h, uid, rank, P: self.lib.fftpde_plan_2d_sharded(
                        ctypes.byref(h), self.nx, self.ny, _DT[dtype], self.Lx, self.Ly, self.device.index, uid,
                        rank, P))
        self.R, self.BW = self.ny // self.P, self.nx // self.P
        self.phys_shape = (self.ny, self.nx) if self.loopback else (self.R, self.nx)
        self.spec_shape = self._lb((self.ny, self.BW))


class ShardedPlan3D(_Sharded):
    """The slab decomposition of an nz x ny x nx volume (fftpde_plan_3d_sharded):
    rank r holds z-planes [r nzl, (r+1) nzl), nzl = nz/P (``phys_shape``
    [nzl, ny, nx]); its spectrum slab is the y-slab, rows [r R, (r+1) R) of all nz
    planes (``spec_shape`` [nz, R, nx]).  One all-to-all each way per transform."""

    def __init__(self, nx: int, ny: int, nz: int, dtype=torch.complex128, Lx: float = 1.0, Ly: float = 1.0,
                 Lz: float = 1.0, device=None, group=None, loopback: int = 0):
        self.nx, self.ny, self.nz = int(nx), int(ny), int(nz)
        self.Lx, self.Ly, self.Lz = float(Lx), float(Ly), float(Lz)
        self._setup(dtype, device, group, loopback,
                    lambda h, uid, rank, P: self.lib.fftpde_plan_3d_sharded(
                        ctypes.byref(h), self.nx, self.ny, self.nz, _DT[dtype], self.Lx, self.Ly, self.Lz,
                        self.device.index, uid, rank, P))
        self.R, self.nzl = self.ny // self.P, self.nz // self.P
        self.phys_shape = (self.nz, self.ny, self.nx) if self.loopback else (self.nzl, self.ny, self.nx)
        self.spec_shape = self._lb((self.nz, self.R, self.nx))


class PencilPlan3D(_Sharded):
    """The pencil decomposition of an nz x ny x nx volume over a pz x py process
    grid (fftpde_plan_3d_pencil): rank r = i py + j holds the
    x-pencil [nz/pz, ny/py, nx] of z-block i and y-block j (``phys_shape``); its
    spectrum is the z-pencil [nz, ny/pz, nx/py] (``spec_shape``).  Two all-to-alls
    per transform, inside the row group (py ranks) and the column group (pz ranks).
    ``loopback=True`` emulates the pz*py ranks in this process: buffers are
    [P, ...] stacks of pencils in rank order."""

    def __init__(self, nx: int, ny: int, nz: int, pz: int, py: int, dtype=torch.complex128, Lx: float = 1.0,
                 Ly: float = 1.0, Lz: float = 1.0, device=None, group=None, loopback: bool = False):
        self.nx, self.ny, self.nz, self.pz, self.py = int(nx), int(ny), int(nz), int(pz), int(py)
        self.Lx, self.Ly, self.Lz = float(Lx), float(Ly), float(Lz)

        def make(h, uid, rank, P):
            if P != self.pz * self.py:
                raise ValueError(f"pencil grid {self.pz} x {self.py} needs {self.pz * self.py} ranks, have {P}")
            return self.lib.fftpde_plan_3d_pencil(ctypes.byref(h), self.nx, self.ny, self.nz, _DT[dtype], self.Lx,
                                                  self.Ly, self.Lz, self.device.index, uid, rank, self.pz, self.py)
        self._setup(dtype, device, group, self.pz * self.py if loopback else 0, make)
        self.phys_shape = self._lb((self.nz // self.pz, self.ny // self.py, self.nx))
        self.spec_shape = self._lb((self.nz, self.ny // self.pz, self.nx // self.py))


class Plan3D(Plan):
    """A 3D plan for [nz, ny, nx] volumes on [0,Lx) x [0,Ly) x [0,Lz) (the n-D
    extension): forward / inverse / poisson / diffuse act on the
    whole volume (fftpde_plan_3d)."""

    def __init__(self, nx: int, ny: int, nz: int, dtype=torch.complex128, Lx: float = 1.0,
                 Ly: float = 1.0, Lz: float = 1.0, device=None):
        if dtype not in _DT:
            raise TypeError("dtype must be torch.complex128 or torch.complex64")
        if not torch.cuda.is_available():
            raise RuntimeError("fftpde needs a CUDA device (no CPU fallback)")
        self.lib = load_library()
        self.device = torch.device(device if device is not None else "cuda")
        if self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        self.nx, self.ny, self.nz, self.dtype = int(nx), int(ny), int(nz), dtype
        self.batch = 1
        self.Lx, self.Ly, self.Lz = float(Lx), float(Ly), float(Lz)
        h = ctypes.c_void_p()
        _check(self.lib.fftpde_plan_3d(ctypes.byref(h), self.nx, self.ny, self.nz, _DT[dtype], self.Lx,
                                       self.Ly, self.Lz, self.device.index), "fftpde_plan_3d")
        self._h = h
        nbytes = self.lib.fftpde_workspace_size(h)
        self.workspace = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=self.device)
        self._bind_stream()
        _check(self.lib.fftpde_set_workspace(h, self.workspace.data_ptr(), self.workspace.numel()),
               "fftpde_set_workspace")

    def _vol(self, x: torch.Tensor, name: str):
        if x.dtype != self.dtype:
            raise TypeError(f"{name}: dtype {x.dtype} does not match the plan's {self.dtype}")
        if tuple(x.shape) != (self.nz, self.ny, self.nx):
            raise ValueError(f"{name}: shape {tuple(x.shape)} does not match plan ({self.nz}, {self.ny}, {self.nx})")

    def _call3(self, fn, x, out, *args):
        self._vol(x, "x")
        xd, host = self._to_dev(x)
        o = self._out(xd, None if host else out)
        self._bind_stream()
        _check(fn(self._h, xd.data_ptr(), o.data_ptr(), *args), fn.__name__)
        return self._finish(o, host, out if host else None)

    def forward(self, x, out=None):
        """3D DFT, + sign, unnormalised (PAPER.md:246-249 extended, :275)."""
        return self._call3(self.lib.fftpde_forward, x, out)

    def inverse(self, X, out=None):
        """3D iDFT, conjugate kernel x 1/(nx ny nz)."""
        return self._call3(self.lib.fftpde_inverse, X, out)

    def poisson(self, rho, out=None):
        """nabla^2 u = rho - mean(rho) in 3D (-1/|k|^2, k = 0 zeroed)."""
        return self._call3(self.lib.fftpde_poisson, rho, out)

    def diffuse(self, u0, D: float, dt: float, nsteps: int, out=None):
        """nsteps exact 3D diffusion steps exp(-D|k|^2 dt)."""
        return self._call3(self.lib.fftpde_diffuse, u0, out, float(D), float(dt), int(nsteps))


_REAL = {torch.float64: (C128, torch.complex128), torch.float32: (C64, torch.complex64)}


class PlanR2C(Plan):
    """A plan for REAL fields [ny, nx] / [B, ny, nx]: Hermitian
    spectra are stored as half spectra [.., ny, nx/2 + 1]; the solves take and return
    real tensors and move half the bytes of the complex path (fftpde_plan_2d_r2c)."""

    def __init__(self, nx: int, ny: int, batch: int = 1, dtype=torch.float64, Lx: float = 1.0,
                 Ly: float = 1.0, device=None):
        if dtype not in _REAL:
            raise TypeError("dtype must be torch.float64 or torch.float32")
        if not torch.cuda.is_available():
            raise RuntimeError("fftpde needs a CUDA device (no CPU fallback)")
        self.lib = load_library()
        self.device = torch.device(device if device is not None else "cuda")
        if self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        self.nx, self.ny, self.batch = int(nx), int(ny), int(batch)
        self.real_dtype, (code, self.dtype) = dtype, _REAL[dtype]
        self.Lx, self.Ly = float(Lx), float(Ly)
        h = ctypes.c_void_p()
        _check(self.lib.fftpde_plan_2d_r2c(ctypes.byref(h), self.nx, self.ny, self.batch, code, self.Lx, self.Ly,
                                           self.device.index), "fftpde_plan_2d_r2c")
        self._h = h
        nbytes = self.lib.fftpde_workspace_size(h)
        self.workspace = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=self.device)
        self._bind_stream()
        _check(self.lib.fftpde_set_workspace(h, self.workspace.data_ptr(), self.workspace.numel()),
               "fftpde_set_workspace")

    def _shape(self, last):
        return ((self.batch,) if self.batch > 1 else ()) + (self.ny, last)

    def _chk(self, x, dtype, last, name):
        if x.dtype != dtype or tuple(x.shape) != self._shape(last):
            raise ValueError(f"{name}: expected {dtype} {self._shape(last)}, got {x.dtype} {tuple(x.shape)}")
        if x.device != self.device or not x.is_contiguous():
            raise ValueError(f"{name}: expected a contiguous tensor on {self.device}")

    def _call(self, fn, x, xdt, xl, odt, ol, out, *args):
        self._chk(x, xdt, xl, "input")
        o = torch.empty(self._shape(ol), dtype=odt, device=self.device) if out is None else out
        self._chk(o, odt, ol, "out")
        self._bind_stream()
        _check(fn(self._h, x.data_ptr(), o.data_ptr(), *args), fn.__name__)
        return o

    def forward(self, x, out=None):
        """Half spectrum X[.., b, a], a <= nx/2, of a real field (+ sign, unnormalised)."""
        return self._call(self.lib.fftpde_forward, x, self.real_dtype, self.nx, self.dtype, self.nx // 2 + 1, out)

    def inverse(self, X, out=None):
        """Real field from its half spectrum (x 1/(nx ny))."""
        return self._call(self.lib.fftpde_inverse, X, self.dtype, self.nx // 2 + 1, self.real_dtype, self.nx, out)

    def poisson(self, rho, out=None):
        return self._call(self.lib.fftpde_poisson, rho, self.real_dtype, self.nx, self.real_dtype, self.nx, out)

    def diffuse(self, u0, D: float, dt: float, nsteps: int, out=None):
        return self._call(self.lib.fftpde_diffuse, u0, self.real_dtype, self.nx, self.real_dtype, self.nx, out,
                          float(D), float(dt), int(nsteps))

    def wave_step(self, u, ut, c: float, dt: float, nsteps: int):
        """In place on the real fields (u, ut)."""
        self._chk(u, self.real_dtype, self.nx, "u")
        self._chk(ut, self.real_dtype, self.nx, "ut")
        self._bind_stream()
        _check(self.lib.fftpde_wave_step(self._h, u.data_ptr(), ut.data_ptr(), float(c), float(dt), int(nsteps)),
               "fftpde_wave_step")
        return u, ut
