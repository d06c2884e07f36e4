"""ctypes binding of the workload generator (include/fracprec_workload.h, libfp_workload.so).

Input side only: synthetic BASELINE systems (restating the reference's mesh.cpp / assembly.cpp) and
snapshot bundles (snapshot.cpp, mmio.cpp).  It does not load the B200 solve library, so the CPU
oracle's callers (bench.py --impl reference, tests) build the same systems without it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "libfp_workload.so")

FP_OK, FP_INVALID_ARGUMENT = 0, 1


class FpCsr(C.Structure):
    _fields_ = [("n_rows", C.c_int32), ("n_cols", C.c_int32),
                ("row_offsets32", C.POINTER(C.c_int32)), ("row_offsets64", C.POINTER(C.c_int64)),
                ("col_indices", C.POINTER(C.c_int32)), ("values", C.POINTER(C.c_double))]


BLOCK_NAMES = ("A", "C1", "Q1", "C2", "H", "Q2", "T", "F_u")


class FpBlockSystem(C.Structure):
    _fields_ = [("n_u", C.c_int32), ("n_t", C.c_int32), ("n_p", C.c_int32)] + [(nm, FpCsr) for nm in BLOCK_NAMES]


class FpFractureSpec(C.Structure):
    _fields_ = [("normal_axis", C.c_int32), ("coord", C.c_double), ("lo1", C.c_double), ("hi1", C.c_double),
                ("lo2", C.c_double), ("hi2", C.c_double)]


class FpWorkloadSpec(C.Structure):
    _fields_ = [("cells", C.c_int32 * 3), ("length", C.c_double * 3), ("n_fractures", C.c_int32),
                ("fractures", C.POINTER(FpFractureSpec)), ("E_median", C.c_double), ("E_sigma_ln", C.c_double),
                ("E_layers", C.c_int32), ("nu", C.c_double), ("nu_lo", C.c_double), ("nu_hi", C.c_double),
                ("frac_stick", C.c_double), ("frac_slip", C.c_double), ("aperture_median", C.c_double),
                ("aperture_sigma_ln", C.c_double), ("seed", C.c_uint64), ("stab_beta", C.c_double),
                ("slip_factor", C.c_double)]


class FpFractureState(C.Structure):
    _fields_ = [("n_p", C.c_int32), ("region", C.c_char_p), ("gap", C.POINTER(C.c_double)),
                ("traction_n", C.POINTER(C.c_double)), ("slip_dir", C.POINTER(C.c_double)),
                ("pressure", C.POINTER(C.c_double))]


_P, _PP, _DP = C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_double)
# every symbol include/fracprec_workload.h declares, with its ctypes signature
SIGNATURES = {
    "fp_workload_last_error": (C.c_char_p, []),
    "fp_workload_layout": (C.c_uint64, []),
    "fp_workload_preset": (C.c_int, [C.c_int32, C.c_uint64, _PP]),
    "fp_workload_custom": (C.c_int, [C.POINTER(FpWorkloadSpec), _PP]),
    "fp_workload_destroy": (None, [_P]),
    "fp_workload_system": (C.c_int, [_P, C.POINTER(FpBlockSystem)]),
    "fp_workload_coords": (C.c_int, [_P, C.POINTER(_DP), C.POINTER(C.c_int32)]),
    "fp_workload_info": (C.c_int, [_P, C.POINTER(C.c_int32)]),
    "fp_workload_region": (C.c_int, [_P, C.POINTER(C.c_char_p), C.POINTER(C.c_double)]),
    "fp_workload_state": (C.c_int, [_P, C.POINTER(FpFractureState)]),
    "fp_workload_set_state": (C.c_int, [_P, C.POINTER(FpFractureState)]),
    "fp_snapshot_import": (C.c_int, [C.c_char_p, _PP]),
    "fp_snapshot_export": (C.c_int, [C.c_char_p, C.POINTER(FpBlockSystem), C.c_char_p, C.c_double, _DP, C.c_int32]),
}


def build() -> None:
    r = subprocess.run(["make", "-j8"], cwd=HERE, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("workload library build failed:\n" + r.stdout[-3000:] + r.stderr[-3000:])


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        build()
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype, fn.argtypes = res, args
    return lib


lib = _load()


def check(status: int) -> None:
    if status == FP_OK:
        return
    msg = (lib.fp_workload_last_error() or b"").decode()
    raise ValueError(msg) if status == FP_INVALID_ARGUMENT else RuntimeError(msg)


@dataclass
class System:
    """A generated (or imported) block system: blocks[name] = (rows, cols, rp int64, ci int32, values)."""
    n_u: int
    n_t: int
    n_p: int
    blocks: dict = field(default_factory=dict)
    node_coords: Optional[np.ndarray] = None

    def total_dimension(self) -> int:
        return self.n_u + self.n_t + self.n_p

    def block_list(self) -> list:
        return [self.blocks[nm] for nm in BLOCK_NAMES]


def system_view(blocks: dict, n_u: int, n_t: int, n_p: int) -> FpBlockSystem:
    """fp_block_system over NumPy CSR tuples (kept alive by the caller)."""
    s = FpBlockSystem()
    s.n_u, s.n_t, s.n_p = n_u, n_t, n_p
    for nm in BLOCK_NAMES:
        r, c, rp, ci, v = blocks[nm]
        m = getattr(s, nm)
        m.n_rows, m.n_cols = r, c
        m.row_offsets64 = rp.ctypes.data_as(C.POINTER(C.c_int64))
        m.col_indices = ci.ctypes.data_as(C.POINTER(C.c_int32))
        m.values = v.ctypes.data_as(C.POINTER(C.c_double))
    return s


class Workload:
    """Synthetic BASELINE config (config_id 1..5 = BASELINE.json configs[0..4]) or a custom spec."""

    def __init__(self, config_id: Optional[int] = None, seed: int = 42, spec: Optional[dict] = None,
                 _handle: Optional[C.c_void_p] = None):
        self._h = C.c_void_p()
        if _handle is not None:
            self._h = _handle
        elif spec is None:
            check(lib.fp_workload_preset(int(config_id), seed, C.byref(self._h)))
        else:
            s = FpWorkloadSpec()
            s.cells[:] = spec["cells"]
            s.length[:] = spec.get("length", (1.0, 1.0, 1.0))
            fr = spec.get("fractures", [])
            arr = (FpFractureSpec * max(1, len(fr)))()
            for i, f in enumerate(fr):
                arr[i] = FpFractureSpec(*f)
            s.n_fractures, s.fractures = len(fr), arr
            s.E_median, s.E_sigma_ln = spec.get("E_median", 10e9), spec.get("E_sigma_ln", 0.0)
            s.E_layers, s.nu = spec.get("E_layers", 0), spec.get("nu", 0.25)
            s.nu_lo, s.nu_hi = spec.get("nu_lo", 0.0), spec.get("nu_hi", 0.0)
            s.frac_stick, s.frac_slip = spec.get("frac_stick", 0.7), spec.get("frac_slip", 0.2)
            s.aperture_median = spec.get("aperture_median", 1e-4)
            s.aperture_sigma_ln = spec.get("aperture_sigma_ln", 0.0)
            s.seed = seed
            s.stab_beta = spec.get("stab_beta", 0.0)
            s.slip_factor = spec.get("slip_factor", 0.0)
            check(lib.fp_workload_custom(C.byref(s), C.byref(self._h)))

    def __del__(self):
        if getattr(self, "_h", None) and lib is not None:
            lib.fp_workload_destroy(self._h)
            self._h = None

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    @classmethod
    def from_snapshot(cls, directory: str) -> "Workload":
        """import_snapshot (snapshot.cpp:67-104): a reference snapshot bundle as a workload."""
        h = C.c_void_p()
        check(lib.fp_snapshot_import(str(directory).encode(), C.byref(h)))
        return cls(_handle=h)

    def region(self) -> tuple:
        """(per-face labels 's'/'l'/'o', dt)"""
        r, dt = C.c_char_p(), C.c_double()
        check(lib.fp_workload_region(self._h, C.byref(r), C.byref(dt)))
        return r.value.decode(), dt.value

    def info(self) -> dict:
        c = (C.c_int32 * 4)()
        check(lib.fp_workload_info(self._h, c))
        return {"stick": c[0], "slip": c[1], "open": c[2], "fractures": c[3]}

    def system(self, copy: bool = True) -> System:
        """The blocks as NumPy CSR tuples: owned copies, or (copy=False) read-only views into the
        workload's arrays (the returned System keeps this Workload alive)."""
        v = FpBlockSystem()
        check(lib.fp_workload_system(self._h, C.byref(v)))

        def arr(p, n):
            a = np.ctypeslib.as_array(p, shape=(n,))
            if copy:
                return a.copy()
            a.flags.writeable = False
            return a

        def take(m: FpCsr):
            if m.n_rows == 0:
                return (0, m.n_cols, np.zeros(1, np.int64), np.zeros(0, np.int32), np.zeros(0))
            rp = arr(m.row_offsets64, m.n_rows + 1)
            nz = int(rp[-1])
            ci = arr(m.col_indices, nz) if nz else np.zeros(0, np.int32)
            vv = arr(m.values, nz) if nz else np.zeros(0)
            return (m.n_rows, m.n_cols, rp, ci, vv)

        xyz = C.POINTER(C.c_double)()
        nn = C.c_int32()
        check(lib.fp_workload_coords(self._h, C.byref(xyz), C.byref(nn)))
        coords = np.ctypeslib.as_array(xyz, shape=(nn.value * 3,)).copy().reshape(-1, 3) if nn.value else None
        S = System(v.n_u, v.n_t, v.n_p, {nm: take(getattr(v, nm)) for nm in BLOCK_NAMES}, coords)
        if not copy:
            S._owner = self
        return S

    def state(self) -> dict:
        """The fracture state (FractureState): region string, gap (n_p x 3), traction_n, slip_dir (n_p x 2),
        pressure — copies."""
        st = FpFractureState()
        check(lib.fp_workload_state(self._h, C.byref(st)))
        n = st.n_p

        def arr(p, k):
            return np.ctypeslib.as_array(p, shape=(n * k,)).copy() if n else np.zeros(0)

        return {"region": st.region.decode()[:n] if n else "", "gap": arr(st.gap, 3).reshape(-1, 3),
                "traction_n": arr(st.traction_n, 1), "slip_dir": arr(st.slip_dir, 2).reshape(-1, 2),
                "pressure": arr(st.pressure, 1)}

    def set_state(self, state: dict) -> None:
        """A new fracture state: C2, H, T, F_u, Q2 re-assembled on the host (assembly.cpp:229-406)."""
        st, keep = state_view(state)
        check(lib.fp_workload_set_state(self._h, C.byref(st)))

    def save_snapshot(self, directory: str) -> None:
        """export_snapshot of this workload (blocks, region labels, dt, node coordinates)."""
        region, dt = self.region()
        S = self.system(copy=False)
        export_snapshot(directory, S.blocks, S.n_u, S.n_t, S.n_p, region, dt, S.node_coords)


def export_snapshot(directory: str, blocks: dict, n_u: int, n_t: int, n_p: int, region: str, dt: float = 0.5,
                    node_coords=None) -> None:
    """export_snapshot (snapshot.cpp:28-65): manifest.json + Matrix Market blocks (+ coords.txt)."""
    keep = {nm: (r, c, np.ascontiguousarray(rp, np.int64), np.ascontiguousarray(ci, np.int32),
                 np.ascontiguousarray(v, np.float64)) for nm, (r, c, rp, ci, v) in blocks.items()}
    view = system_view(keep, n_u, n_t, n_p)
    coords = None if node_coords is None else np.ascontiguousarray(node_coords, dtype=np.float64)
    cp = coords.ctypes.data_as(C.POINTER(C.c_double)) if coords is not None else None
    nn = 0 if coords is None else coords.shape[0]
    check(lib.fp_snapshot_export(str(directory).encode(), C.byref(view), region.encode(), float(dt), cp, nn))


def state_view(state: dict):
    """(fp_fracture_state over NumPy copies of a state dict, keepalive)."""
    region = state["region"].encode()
    gap = np.ascontiguousarray(state["gap"], np.float64).reshape(-1)
    tn = np.ascontiguousarray(state["traction_n"], np.float64)
    sd = np.ascontiguousarray(state["slip_dir"], np.float64).reshape(-1)
    pr = np.ascontiguousarray(state["pressure"], np.float64)
    st = FpFractureState()
    st.n_p = len(region)
    st.region = region
    st.gap, st.traction_n = gap.ctypes.data_as(_DP), tn.ctypes.data_as(_DP)
    st.slip_dir, st.pressure = sd.ctypes.data_as(_DP), pr.ctypes.data_as(_DP)
    return st, (region, gap, tn, sd, pr)
