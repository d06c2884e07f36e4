"""Python host mirror of the reference's solve-path API over the C ABI.

Names and argument meaning follow /root/reference/proj/core/include/fracprec/:
``CsrMatrix`` (csr.hpp:16-49), ``BlockSystem`` (block.hpp:36-45),
``AmgConfig`` (amg.hpp:19-31), ``PrecondConfig`` (precond.hpp:19-30),
``build_tpu`` / ``build_tup`` (precond.hpp:76-85), ``TpuOperator`` /
``TupOperator`` (precond.hpp:94-116), ``BlockSystemOperator`` (block.hpp:48-57),
``gmres`` (gmres.hpp:29-33) and ``SolveStats`` (gmres.hpp:15-22).  Errors raise
``ValueError`` (std::invalid_argument) or ``NumericalError``.

Vectors may be NumPy arrays (host memory, copied through the ABI) or CUDA
torch tensors (device memory, used in place).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _native as N
from workload import gen as _wl  # the input-side generator library (loaded with the solve library)
from ._native import NumericalError  # noqa: F401  (re-export)

_VARIANTS = {"tpu": N.FP_TPU, "tup": N.FP_TUP, "tup_star": N.FP_TUP_STAR}


@dataclass
class CsrMatrix:
    n_rows: int
    n_cols: int
    row_offsets: np.ndarray
    col_indices: np.ndarray
    values: np.ndarray

    def __post_init__(self):
        self.row_offsets = np.ascontiguousarray(self.row_offsets, dtype=np.int64)
        self.col_indices = np.ascontiguousarray(self.col_indices, dtype=np.int32)
        self.values = np.ascontiguousarray(self.values, dtype=np.float64)

    @property
    def nnz(self) -> int:
        return int(self.row_offsets[-1]) if self.n_rows > 0 else 0

    @staticmethod
    def empty(rows: int, cols: int) -> "CsrMatrix":
        return CsrMatrix(rows, cols, np.zeros(rows + 1, np.int64), np.zeros(0, np.int32), np.zeros(0))

    def view(self) -> N.FpCsr:
        v = N.FpCsr()
        v.n_rows, v.n_cols = self.n_rows, self.n_cols
        v.row_offsets64 = self.row_offsets.ctypes.data_as(C.POINTER(C.c_int64))
        v.col_indices = self.col_indices.ctypes.data_as(C.POINTER(C.c_int32))
        v.values = self.values.ctypes.data_as(C.POINTER(C.c_double))
        return v

    def matvec(self, x: np.ndarray) -> np.ndarray:  # host helper for checks (not on the solve path)
        rows = np.repeat(np.arange(self.n_rows), np.diff(self.row_offsets))
        y = np.zeros(self.n_rows)
        np.add.at(y, rows, self.values * x[self.col_indices])
        return y


@dataclass
class BlockSystem:
    n_u: int
    n_t: int
    n_p: int
    A: CsrMatrix
    C1: CsrMatrix
    Q1: CsrMatrix
    C2: CsrMatrix
    H: CsrMatrix
    Q2: CsrMatrix
    T: CsrMatrix
    F_u: Optional[CsrMatrix] = None
    node_coords: Optional[np.ndarray] = None  # (n_nodes, 3) for the rigid-body near-null space

    def total_dimension(self) -> int:
        return self.n_u + self.n_t + self.n_p

    def view(self) -> N.FpBlockSystem:
        s = N.FpBlockSystem()
        s.n_u, s.n_t, s.n_p = self.n_u, self.n_t, self.n_p
        for nm in ("A", "C1", "Q1", "C2", "H", "Q2", "T"):
            setattr(s, nm, getattr(self, nm).view())
        s.F_u = (self.F_u or CsrMatrix.empty(0, self.n_u)).view()
        return s


@dataclass
class AmgConfig:
    strength_threshold: float = 0.08
    max_coarse: int = 100
    pre_sweeps: int = 1
    post_sweeps: int = 1
    # "weighted_jacobi" (reference option), "sgs" (reference default; no GPU path), or the extensions
    # of SURVEY §8(f) item 4, both restated in the oracle: "chebyshev" (degree-k Chebyshev in D^-1 A)
    # and "multicolor_gs" (symmetric Gauss-Seidel visiting rows colour by colour, greedy colouring)
    smoother: str = "weighted_jacobi"
    prolongation_smoothing: bool = True
    cycles_per_apply: int = 1
    jacobi_omega: float = 2.0 / 3.0
    stall_ratio: float = 0.9
    max_levels: int = 25
    chebyshev_degree: int = 2
    chebyshev_ratio: float = 10.0
    power_iterations: int = 10
    # "ordered" (the reference's summation order) or "strided" (extension: coarse operators summed
    # as 32 lane-strided partials + xor tree, one warp per row; restated in the oracle)
    row_sum: str = "ordered"

    _SMOOTHERS = {"weighted_jacobi": 0, "sgs": 1, "chebyshev": 2, "multicolor_gs": 3}
    _ROW_SUMS = {"ordered": 0, "strided": 1}

    def native(self) -> N.FpAmgConfig:
        if self.smoother not in self._SMOOTHERS:
            raise ValueError(f"unknown smoother {self.smoother!r}")
        c = N.FpAmgConfig()
        c.strength_threshold, c.max_coarse = self.strength_threshold, self.max_coarse
        c.pre_sweeps, c.post_sweeps = self.pre_sweeps, self.post_sweeps
        c.smoother = self._SMOOTHERS[self.smoother]
        c.prolongation_smoothing = int(self.prolongation_smoothing)
        c.cycles_per_apply, c.jacobi_omega = self.cycles_per_apply, self.jacobi_omega
        c.stall_ratio, c.max_levels = self.stall_ratio, self.max_levels
        c.chebyshev_degree, c.chebyshev_ratio = self.chebyshev_degree, self.chebyshev_ratio
        c.power_iterations = self.power_iterations
        if self.row_sum not in self._ROW_SUMS:
            raise ValueError(f"unknown row_sum {self.row_sum!r} (ordered | strided)")
        c.row_sum = self._ROW_SUMS[self.row_sum]
        return c


_FACTOR_SOLVE = {"auto": 0, "sweep": 1, "inverse": 2, "panel": 3}


def _factor_mode(name: str) -> int:
    if name not in _FACTOR_SOLVE:
        raise ValueError(f"unknown factor_solve {name!r} (auto | sweep | inverse | panel)")
    return _FACTOR_SOLVE[name]


@dataclass
class PrecondConfig:
    variant: str = "tup"
    inner: str = "amg"
    amg: AmgConfig = field(default_factory=AmgConfig)
    # how T / S~2 (SparseFactor) is applied: "sweep", "inverse" (explicit block
    # inverses streamed from HBM) or "auto" (the faster that fits)
    factor_solve: str = "auto"

    def native(self) -> N.FpPrecondConfig:
        if self.inner != "amg":
            raise ValueError("the GPU path implements inner = amg only")
        if self.variant not in _VARIANTS:
            raise ValueError(f"unknown variant {self.variant!r}")
        c = N.FpPrecondConfig()
        c.variant = _VARIANTS[self.variant]
        c.amg = self.amg.native()
        c.factor_solve = _factor_mode(self.factor_solve)
        return c


@dataclass
class SolveStats:
    iterations: int = 0
    relative_residuals: list = field(default_factory=list)
    converged: bool = False
    breakdown: bool = False
    restarts: int = 0
    precond_applies: int = 0
    device_seconds: float = 0.0
    kernel_launches: int = 0
    probe_ms: float = 0.0      # probe=True: summed CUDA-event time of the finest-level Jacobi sweeps
    probe_launches: int = 0
    reorth_steps: int = 0      # Arnoldi steps that ran the DGKS second pass (gmres.cpp:96-102)


def _vec(x, n: int):
    """(pointer, mem kind, keepalive) for an input vector: a NumPy array or a CUDA tensor of length n.

    The library runs on its own non-blocking stream, so before a device pointer is handed over the
    producing torch stream is synchronized (the ABI call returns only after its results are written;
    include/fracprec_b200.h states the ordering contract)."""
    if hasattr(x, "is_cuda") and x.is_cuda:
        import torch

        if x.dtype != torch.float64 or not x.is_contiguous() or x.numel() != n:
            raise ValueError("device vectors must be contiguous float64 tensors of the operator dimension")
        torch.cuda.current_stream(x.device).synchronize()
        return C.c_void_p(x.data_ptr()), N.FP_MEM_DEVICE, x
    a = np.ascontiguousarray(x, dtype=np.float64)
    if a.size != n:
        raise ValueError(f"dimension mismatch: expected {n}, got {a.size}")
    return C.c_void_p(a.ctypes.data), N.FP_MEM_HOST, a


def _out(y, n: int):
    """(pointer, mem kind, keepalive) for an output vector, written in place: a writeable C-contiguous
    float64 NumPy array or a contiguous float64 CUDA tensor of length n (no silent temporary copy)."""
    if hasattr(y, "is_cuda") and y.is_cuda:
        return _vec(y, n)
    if not (isinstance(y, np.ndarray) and y.dtype == np.float64 and y.flags.c_contiguous and y.flags.writeable):
        raise ValueError("output vectors must be writeable C-contiguous float64 arrays (or CUDA float64 tensors)")
    if y.size != n:
        raise ValueError(f"dimension mismatch: expected {n}, got {y.size}")
    return C.c_void_p(y.ctypes.data), N.FP_MEM_HOST, y


def _out_like(x, n: int):
    if hasattr(x, "is_cuda") and x.is_cuda:
        import torch

        return torch.empty(n, dtype=torch.float64, device=x.device)
    return np.empty(n)


class BlockSystemOperator:
    """Device-resident J; ``apply`` is BlockSystemOperator::apply (block.cpp:70-74)."""

    def __init__(self, J: BlockSystem):
        self.J = J
        self._h = C.c_void_p()
        N.check(N.lib.fp_system_create(C.byref(J.view()), C.byref(self._h)))
        self._n = J.total_dimension()

    def __del__(self):
        if getattr(self, "_h", None) and N is not None and getattr(N, "lib", None) is not None:
            N.lib.fp_system_destroy(self._h)
            self._h = None

    def dimension(self) -> int:
        return self._n

    def apply(self, x, y=None):
        y = _out_like(x, self._n) if y is None else y
        xp, mem, _ka = _vec(x, self._n)
        yp, mem2, _kb = _out(y, self._n)
        if mem != mem2:
            raise ValueError("x and y must live in the same memory space")
        N.check(N.lib.fp_system_apply(self._h, xp, yp, mem))
        return y

    __call__ = apply

    def block_scaling(self):
        st, sp = C.c_double(), C.c_double()
        N.check(N.lib.fp_block_scaling(self._h, C.byref(st), C.byref(sp)))
        return st.value, sp.value


class HostPreconditioner:
    """Host-built preconditioner data (build_tpu / build_tup, precond.cpp:119-202)."""

    def __init__(self, J: Optional[BlockSystem], cfg: PrecondConfig, _workload: "Optional[Workload]" = None):
        self._h = C.c_void_p()
        self.variant = cfg.variant
        if _workload is not None:  # from_workload: no copy of the blocks
            N.check(N.lib.fp_workload_host_precond_build(_workload._h, C.byref(cfg.native()), C.byref(self._h)))
            return
        coords = None if J.node_coords is None else np.ascontiguousarray(J.node_coords, dtype=np.float64)
        cp = coords.ctypes.data_as(C.POINTER(C.c_double)) if coords is not None else None
        nn = 0 if coords is None else coords.shape[0]
        N.check(N.lib.fp_host_precond_build(C.byref(J.view()), C.byref(cfg.native()), cp, nn, C.byref(self._h)))

    @classmethod
    def from_workload(cls, W: "Workload", cfg: PrecondConfig) -> "HostPreconditioner":
        """build_tpu / build_tup on a generated workload in place (fp_workload_host_precond_build)."""
        return cls(None, cfg, _workload=W)

    def __del__(self):
        if getattr(self, "_h", None) and N is not None and getattr(N, "lib", None) is not None:
            N.lib.fp_host_precond_destroy(self._h)
            self._h = None

    def set_upload(self, row_sum: str, factor_solve: str = "auto") -> None:
        """Upload-time choices for the next GpuPreconditioner.from_host: coarse row-sum order
        ("ordered" | "strided") and factor application ("auto" | "sweep" | "inverse")."""
        if row_sum not in AmgConfig._ROW_SUMS:
            raise ValueError(f"unknown row_sum {row_sum!r} (ordered | strided)")
        N.check(N.lib.fp_host_precond_set_upload(self._h, AmgConfig._ROW_SUMS[row_sum], _factor_mode(factor_solve)))

    def level_sizes(self) -> list:
        nl = C.c_int32()
        N.check(N.lib.fp_host_precond_levels(self._h, C.byref(nl), None))
        rows = (C.c_int32 * nl.value)()
        N.check(N.lib.fp_host_precond_levels(self._h, None, rows))
        return list(rows)

    def matrix(self, what: int, level: int = 0) -> CsrMatrix:
        r, c, nz = C.c_int32(), C.c_int32(), C.c_int64()
        N.check(N.lib.fp_host_precond_matrix(self._h, what, level, C.byref(r), C.byref(c), C.byref(nz), None, None, None))
        rp = np.zeros(r.value + 1, np.int64)
        ci = np.zeros(nz.value, np.int32)
        v = np.zeros(nz.value)
        N.check(N.lib.fp_host_precond_matrix(
            self._h, what, level, None, None, None, rp.ctypes.data_as(C.POINTER(C.c_int64)),
            ci.ctypes.data_as(C.POINTER(C.c_int32)), v.ctypes.data_as(C.POINTER(C.c_double))))
        return CsrMatrix(r.value, c.value, rp, ci, v)

    def vector(self, what: int, level: int = 0) -> np.ndarray:
        n = C.c_int64()
        N.check(N.lib.fp_host_precond_vector(self._h, what, level, None, C.byref(n)))
        out = np.zeros(n.value)
        N.check(N.lib.fp_host_precond_vector(self._h, what, level, out.ctypes.data_as(C.POINTER(C.c_double)), None))
        return out


class GpuPreconditioner:
    """Device-resident M^-1; ``apply`` is TpuOperator / TupOperator::apply (precond.cpp:285-296)."""

    def __init__(self, op: BlockSystemOperator, handle: C.c_void_p, variant: str):
        self.op, self._h, self.variant = op, handle, variant
        self._n = op.dimension()

    @classmethod
    def from_host(cls, op: BlockSystemOperator, hp: HostPreconditioner) -> "GpuPreconditioner":
        h = C.c_void_p()
        N.check(N.lib.fp_precond_create(op._h, hp._h, C.byref(h)))
        return cls(op, h, hp.variant)

    @classmethod
    def upload(cls, op: BlockSystemOperator, variant: str, h_blocks: np.ndarray, factor_matrix: CsrMatrix,
               levels: Sequence[tuple], amg: AmgConfig, factor_solve: str = "auto") -> "GpuPreconditioner":
        """Upload a reference-built hierarchy: levels = [(A_l, P_l or None, smoother_diag_l), ...]."""
        keep = []
        descs = (N.FpAmgLevelDesc * len(levels))()
        for i, (A, P, d) in enumerate(levels):
            d = np.ascontiguousarray(d, dtype=np.float64)
            keep.append(d)
            descs[i].A = A.view()
            descs[i].P = (P if P is not None else CsrMatrix.empty(0, 0)).view()
            descs[i].smoother_diag = d.ctypes.data_as(C.POINTER(C.c_double))
        hb = np.ascontiguousarray(h_blocks, dtype=np.float64)
        desc = N.FpPrecondDesc()
        desc.variant = _VARIANTS[variant]
        desc.h_blocks = hb.ctypes.data_as(C.POINTER(C.c_double))
        desc.factor_matrix = factor_matrix.view()
        desc.n_levels = len(levels)
        desc.levels = descs
        desc.amg = amg.native()
        desc.factor_solve = _factor_mode(factor_solve)
        h = C.c_void_p()
        N.check(N.lib.fp_precond_upload(op._h, C.byref(desc), C.byref(h)))
        return cls(op, h, variant)

    def __del__(self):
        if getattr(self, "_h", None) and N is not None and getattr(N, "lib", None) is not None:
            N.lib.fp_precond_destroy(self._h)
            self._h = None

    def dimension(self) -> int:
        return self._n

    def apply(self, x, y=None):
        y = _out_like(x, self._n) if y is None else y
        xp, mem, _ka = _vec(x, self._n)
        yp, mem2, _kb = _out(y, self._n)
        if mem != mem2:
            raise ValueError("x and y must live in the same memory space")
        N.check(N.lib.fp_precond_apply(self._h, xp, yp, mem))
        return y

    __call__ = apply

    def amg_apply(self, r):
        n_u = self.op.J.n_u
        x = _out_like(r, n_u)
        rp, mem, _ka = _vec(r, n_u)
        xp, _m, _kb = _out(x, n_u)
        N.check(N.lib.fp_amg_apply(self._h, rp, xp, mem))
        return x

    @property
    def factor_solve(self) -> str:
        """The factor application this preconditioner resolved to: 'sweep', 'inverse' or 'panel'."""
        m = C.c_int32()
        N.check(N.lib.fp_precond_factor_solve(self._h, C.byref(m)))
        return {1: "sweep", 2: "inverse", 3: "panel"}[m.value]

    def call_count(self) -> int:
        return int(N.lib.fp_precond_inner_calls(self._h, 0))

    def reset_count(self) -> None:
        N.lib.fp_precond_inner_calls(self._h, 1)

    def profile(self, reps: int = 20) -> dict:
        """Per-phase CUDA-event timings (ms per launch) and algorithmic bytes (fp_precond_profile)."""
        p = N.FpProfile()
        N.check(N.lib.fp_precond_profile(self._h, reps, C.byref(p)))
        arrays = ("level_rows", "level_nnz", "vcycle_ms")
        out = {k: getattr(p, k) for k, _ in N.FpProfile._fields_ if k not in arrays}
        for k in arrays:
            out[k] = list(getattr(p, k)[: p.n_levels])
        return out

    def traffic(self):
        ab, jb, la = C.c_double(), C.c_double(), C.c_int32()
        N.check(N.lib.fp_precond_traffic(self._h, C.byref(ab), C.byref(la), C.byref(jb)))
        return {"apply_bytes": ab.value, "apply_launches": la.value, "japply_bytes": jb.value}


def _build(J: BlockSystem, cfg: PrecondConfig, op: Optional[BlockSystemOperator]):
    op = op or BlockSystemOperator(J)
    return GpuPreconditioner.from_host(op, HostPreconditioner(J, cfg))


def build_tpu(J: BlockSystem, cfg: Optional[PrecondConfig] = None, op: Optional[BlockSystemOperator] = None):
    cfg = cfg or PrecondConfig()
    cfg.variant = "tpu"
    return _build(J, cfg, op)


def build_tup(J: BlockSystem, cfg: Optional[PrecondConfig] = None, op: Optional[BlockSystemOperator] = None,
              star: bool = False):
    cfg = cfg or PrecondConfig()
    cfg.variant = "tup_star" if star else "tup"
    return _build(J, cfg, op)


def gmres(op: BlockSystemOperator, precond: GpuPreconditioner, b, tol: float, max_iter: int = 500,
          restart: Optional[int] = None, scaled: bool = False, x=None, orthogonalization: str = "mgs",
          probe: bool = False):
    """Right-preconditioned GMRES, x0 = 0 (gmres.hpp:29-33); ``restart`` gives GMRES(m);
    ``scaled`` solves the driver's D J D system with D^-1 M D^-1 (driver.cpp:229-255);
    ``orthogonalization`` "mgs" (the reference's loop) or "cgs" (classical, one reduction
    per pass, same DGKS second-pass test); ``probe`` times the finest-level Jacobi sweep of
    every Arnoldi step with CUDA events inside the graph (stats.probe_ms / probe_launches)."""
    n = op.dimension()
    x = _out_like(b, n) if x is None else x
    bp, mem, _ka = _vec(b, n)
    xp, mem_x, _kb = _out(x, n)
    if mem != mem_x:
        raise ValueError("gmres: b and x must live in the same memory space")
    o = N.FpGmresOptions()
    if orthogonalization not in ("mgs", "cgs"):
        raise ValueError("gmres: orthogonalization must be 'mgs' or 'cgs'")
    o.tol, o.restart, o.max_iter, o.scaled = tol, restart or max_iter, max_iter, int(scaled)
    o.orthogonalization = 1 if orthogonalization == "cgs" else 0
    o.probe = int(probe)
    hist = np.zeros(max(1, max_iter))
    st = N.FpSolveStats()
    st.residual_history = hist.ctypes.data_as(C.POINTER(C.c_double))
    st.history_capacity = hist.size
    N.check(N.lib.fp_gmres(op._h, precond._h, bp, xp, mem, C.byref(o), C.byref(st)))
    stats = SolveStats(st.iterations, list(hist[: st.history_len]), bool(st.converged), bool(st.breakdown),
                       st.restarts, st.precond_applies, st.device_seconds, int(st.kernel_launches), st.probe_ms,
                       st.probe_launches, st.reorth_steps)
    return x, stats


# ----------------------------------------------------------------- workloads
def _csr(t) -> CsrMatrix:
    r, c, rp, ci, v = t
    return CsrMatrix(r, c, rp, ci, v)


class Workload:
    """Synthetic BASELINE config (include/fracprec_workload.h): the generator library's workload
    (workload/gen.py) with its blocks as this API's BlockSystem."""

    def __init__(self, config_id: Optional[int] = None, seed: int = 42, spec: Optional[dict] = None,
                 _gen: "Optional[_wl.Workload]" = None):
        self._w = _gen if _gen is not None else _wl.Workload(config_id, seed, spec)

    @property
    def _h(self):
        return self._w.handle

    @classmethod
    def from_snapshot(cls, directory: str) -> "Workload":
        """import_snapshot (snapshot.cpp:67-104): a reference snapshot bundle as a workload."""
        return cls(_gen=_wl.Workload.from_snapshot(directory))

    def region(self) -> tuple:
        """(per-face labels 's'/'l'/'o', dt)"""
        return self._w.region()

    def save_snapshot(self, directory: str) -> None:
        """export_snapshot of this workload (blocks, region labels, dt, node coordinates)."""
        self._w.save_snapshot(directory)

    def info(self) -> dict:
        return self._w.info()

    def state(self) -> dict:
        """The fracture state (region, gap, traction_n, slip_dir, pressure)."""
        return self._w.state()

    def set_state(self, state: dict) -> None:
        """A new fracture state, the blocks re-assembled on the host (the reference's Newton-step assembly)."""
        self._w.set_state(state)

    def system(self, copy: bool = True) -> BlockSystem:
        """The generated blocks as a BlockSystem: owned NumPy copies, or (copy=False) read-only
        views into the workload's arrays that keep the Workload alive."""
        S = self._w.system(copy=copy)
        blocks = {nm: _csr(t) for nm, t in S.blocks.items()}
        J = BlockSystem(S.n_u, S.n_t, S.n_p, node_coords=S.node_coords, **blocks)
        if not copy:
            J._owner = self  # the views point into this workload
        return J


class FractureAssembly:
    """assemble_fracture_blocks (assembly.cpp:229-406) on the device: C2, H, T, F_u, Q2 for a fracture state,
    optionally installed into a BlockSystemOperator (the Newton step's re-assembly; fp_fracture_assembly_*)."""

    BLOCKS = ("C2", "H", "T", "F_u", "Q2")

    def __init__(self, W: Workload):
        self._h = C.c_void_p()
        self._w = W
        N.check(N.lib.fp_fracture_assembly_create(W._h, C.byref(self._h)))

    def __del__(self):
        if getattr(self, "_h", None) and N is not None and getattr(N, "lib", None) is not None:
            N.lib.fp_fracture_assembly_destroy(self._h)
            self._h = None

    def run(self, state: dict, op: Optional[BlockSystemOperator] = None) -> None:
        st, _keep = _wl.state_view(state)
        N.check(N.lib.fp_fracture_assembly_run(self._h, C.byref(st), op._h if op is not None else None))

    def matrix(self, name: str) -> CsrMatrix:
        what = self.BLOCKS.index(name)
        r, c, nz = C.c_int32(), C.c_int32(), C.c_int64()
        N.check(N.lib.fp_fracture_assembly_matrix(self._h, what, C.byref(r), C.byref(c), C.byref(nz), None, None, None))
        rp, ci, v = np.zeros(r.value + 1, np.int64), np.zeros(nz.value, np.int32), np.zeros(nz.value)
        N.check(N.lib.fp_fracture_assembly_matrix(
            self._h, what, None, None, None, rp.ctypes.data_as(C.POINTER(C.c_int64)),
            ci.ctypes.data_as(C.POINTER(C.c_int32)), v.ctypes.data_as(C.POINTER(C.c_double))))
        return CsrMatrix(r.value, c.value, rp, ci, v)


def export_snapshot(directory: str, J: BlockSystem, region: str, dt: float = 0.5) -> None:
    """export_snapshot (snapshot.cpp:28-65): manifest.json + Matrix Market blocks (+ coords.txt)."""
    blocks = {nm: (m.n_rows, m.n_cols, m.row_offsets, m.col_indices, m.values)
              for nm, m in zip(_wl.BLOCK_NAMES, (J.A, J.C1, J.Q1, J.C2, J.H, J.Q2, J.T,
                                                 J.F_u or CsrMatrix.empty(0, J.n_u)))}
    _wl.export_snapshot(directory, blocks, J.n_u, J.n_t, J.n_p, region, dt, J.node_coords)


def set_setup_backend(where: str) -> None:
    """Where build_tpu / build_tup run: "device" (csrc/device/dsetup.cu: the fine-size products, strength
    graph and Galerkin products in HBM; the default with a CUDA device) or "host" (OpenMP, setup.cpp).
    Both build the oracle's hierarchy bit for bit."""
    N.check(N.lib.fp_set_setup_backend(1 if where == "device" else 0))


def setup_backend() -> str:
    """Where the preconditioner setup runs: "device" (default with a CUDA device) or "host"."""
    d = C.c_int32()
    N.check(N.lib.fp_setup_backend(C.byref(d)))
    return "device" if d.value else "host"
