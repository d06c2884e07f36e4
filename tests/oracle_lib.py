"""ctypes driver of the CPU oracle (oracle/, TEST INFRASTRUCTURE ONLY).

Used by tests/ as the checker, by __graft_entry__.smoke() and by bench.py's
cpu_baseline / --impl reference legs.  Nothing in the product imports this.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
LIB = os.path.join(ORACLE_DIR, "_build", "liboracle.so")
KAT = os.path.join(ORACLE_DIR, "_build", "oracle_kat")


def build() -> None:
    r = subprocess.run(["make", "-j8"], cwd=ORACLE_DIR, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + r.stdout[-3000:] + r.stderr[-3000:])


def _load():
    if not os.path.exists(LIB) and os.path.exists(os.path.join(ORACLE_DIR, "Makefile")):
        build()
    lib = C.CDLL(LIB)
    P, PP, DP, IP = C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_double), C.POINTER(C.c_int)
    sig = {
        "or_last_error": (C.c_char_p, []),
        "or_set_threads": (None, [C.c_int]),
        "or_threads": (C.c_int, []),
        "or_set_chunked_reductions": (None, [C.c_int]),
        "or_system_create": (C.c_int, [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p),
                                       C.POINTER(C.c_void_p), IP, IP, PP]),
        "or_system_toy": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_uint, PP]),
        "or_system_destroy": (None, [P]),
        "or_system_dims": (C.c_int, [P, IP, IP, IP]),
        "or_system_block": (P, [P, C.c_int]),
        "or_system_apply": (C.c_int, [P, DP, DP]),
        "or_csr_info": (C.c_int, [P, IP, IP, C.POINTER(C.c_int64)]),
        "or_csr_copy": (C.c_int, [P, C.POINTER(C.c_int64), IP, DP]),
        "or_precond_build": (C.c_int, [P, C.c_int, C.c_int, DP, IP, DP, C.c_int, PP]),
        "or_precond_set_factor_solve": (C.c_int, [P, C.c_int]),
        "or_precond_factor_pivots": (C.c_int, [P]),
        "or_precond_set_row_sum": (C.c_int, [P, C.c_int]),
        "or_precond_destroy": (None, [P]),
        "or_precond_apply": (C.c_int, [P, DP, DP]),
        "or_precond_inner_calls": (C.c_long, [P, C.c_int]),
        "or_precond_matrix": (P, [P, C.c_int]),
        "or_precond_hblocks": (C.c_int, [P, DP]),
        "or_precond_vec": (C.c_int, [P, C.c_int, DP]),
        "or_amg_levels": (C.c_int, [P]),
        "or_amg_level_matrix": (P, [P, C.c_int, C.c_int]),
        "or_amg_level_diag": (C.c_int, [P, C.c_int, DP]),
        "or_amg_level_lambda": (C.c_double, [P, C.c_int]),
        "or_amg_level_aggregates": (C.c_int, [P, C.c_int, IP]),
        "or_amg_apply": (C.c_int, [P, DP, DP]),
        "or_amg_level_colors": (C.c_int, [P, C.c_int, IP, IP]),
        "or_gmres": (C.c_int, [P, P, DP, C.c_double, C.c_int, C.c_int, C.c_int, DP, IP, DP, C.c_int, DP]),
        "or_block_scaling": (C.c_int, [P, DP]),
        "or_mm_read": (C.c_int, [C.c_char_p, PP]),
        "or_csr_destroy": (None, [P]),
        "or_mm_write": (C.c_int, [C.c_char_p, C.c_int, C.c_int, C.POINTER(C.c_int64), IP, DP]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype, f.argtypes = res, args
    return lib


lib = _load()


def set_threads(n: int) -> None:
    """Threads of the oracle's independent row / block / aggregate loops (oracle/par.hpp); every
    result is bitwise independent of it.  Reductions stay sequential."""
    lib.or_set_threads(int(n))


def threads() -> int:
    return int(lib.or_threads())


def set_chunked_reductions(on: bool) -> None:
    """GMRES dots / norms as fixed 32768-entry chunk sums (threaded, deterministic) instead of the
    reference's single left-to-right sum: a different rounding of the same algorithm."""
    lib.or_set_chunked_reductions(int(bool(on)))


# the checker runs on every host core; the timed CPU legs of bench.py choose their own count
set_threads(int(os.environ.get("FRACPREC_ORACLE_THREADS", os.cpu_count() or 1)))


def _check(st: int) -> None:
    if st != 0:
        msg = lib.or_last_error().decode()
        if st == 1:
            raise ValueError(msg)
        raise RuntimeError(f"oracle error {st}: {msg}")


def _dp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def csr_from(handle) -> tuple:
    """(n_rows, n_cols, row_offsets int64, col_indices int32, values)"""
    r, c, nz = C.c_int(), C.c_int(), C.c_int64()
    _check(lib.or_csr_info(handle, C.byref(r), C.byref(c), C.byref(nz)))
    rp = np.zeros(r.value + 1, np.int64)
    ci = np.zeros(nz.value, np.int32)
    v = np.zeros(nz.value)
    lib.or_csr_copy(handle, rp.ctypes.data_as(C.POINTER(C.c_int64)), ci.ctypes.data_as(C.POINTER(C.c_int)), _dp(v))
    return r.value, c.value, rp, ci, v


AMG_DEFAULT = dict(strength_threshold=0.08, jacobi_omega=2.0 / 3.0, stall_ratio=0.9, max_coarse=100, pre_sweeps=1,
                   post_sweeps=1, smoother=0, prolongation_smoothing=1, cycles_per_apply=1, max_levels=25,
                   chebyshev_degree=2, chebyshev_ratio=10.0, power_iterations=10)
VARIANT = {"tpu": 0, "tup": 1, "tup_star": 2}


class OracleSystem:
    def __init__(self, handle):
        self.h = handle
        nu, nt, np_ = C.c_int(), C.c_int(), C.c_int()
        lib.or_system_dims(self.h, C.byref(nu), C.byref(nt), C.byref(np_))
        self.n_u, self.n_t, self.n_p = nu.value, nt.value, np_.value
        self.n = self.n_u + self.n_t + self.n_p

    @classmethod
    def toy(cls, n_u, n_p, mode, seed=99):
        modes = {"decoupled": 0, "stick": 1, "mixed": 2, "open_all": 3}
        h = C.c_void_p()
        _check(lib.or_system_toy(n_u, n_p, modes[mode], seed, C.byref(h)))
        return cls(h)

    @classmethod
    def from_blocks(cls, n_u, n_t, n_p, blocks):
        """blocks: 8 tuples (rows, cols, rp int64, ci int32, v) in order A, C1, Q1, C2, H, Q2, T, F_u."""
        keep = []
        rps, cis, vs = (C.c_void_p * 8)(), (C.c_void_p * 8)(), (C.c_void_p * 8)()
        rows, cols = (C.c_int * 8)(), (C.c_int * 8)()
        for i, (r, c, rp, ci, v) in enumerate(blocks):
            rp = np.ascontiguousarray(rp, np.int64)
            ci = np.ascontiguousarray(ci, np.int32)
            v = np.ascontiguousarray(v, np.float64)
            keep += [rp, ci, v]
            rps[i], cis[i], vs[i] = rp.ctypes.data, ci.ctypes.data, v.ctypes.data
            rows[i], cols[i] = r, c
        h = C.c_void_p()
        _check(lib.or_system_create(n_u, n_t, n_p, rps, cis, vs, rows, cols, C.byref(h)))
        return cls(h)

    def __del__(self):
        if getattr(self, "h", None) and lib is not None:
            lib.or_system_destroy(self.h)
            self.h = None

    def block(self, which: int) -> tuple:
        return csr_from(lib.or_system_block(self.h, which))

    def blocks(self) -> list:
        return [self.block(i) for i in range(8)]

    def apply(self, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float64)
        y = np.zeros(self.n)
        _check(lib.or_system_apply(self.h, _dp(x), _dp(y)))
        return y

    def scaling(self):
        out = np.zeros(2)
        lib.or_block_scaling(self.h, _dp(out))
        return float(out[0]), float(out[1])


class OraclePrecond:
    def __init__(self, sys: OracleSystem, variant="tup", inner="amg", coords=None, factor_solve="sweep",
                 row_sum="ordered", **amg):
        cfg = dict(AMG_DEFAULT, **amg)
        d = np.array([cfg["strength_threshold"], cfg["jacobi_omega"], cfg["stall_ratio"], cfg["chebyshev_ratio"]])
        i = np.array([cfg["max_coarse"], cfg["pre_sweeps"], cfg["post_sweeps"], cfg["smoother"],
                      cfg["prolongation_smoothing"], cfg["cycles_per_apply"], cfg["max_levels"],
                      cfg["chebyshev_degree"], cfg["power_iterations"]], np.int32)
        self.sys, self.variant = sys, variant
        self.h = C.c_void_p()
        cp, nn = None, 0
        if coords is not None:
            self._coords = np.ascontiguousarray(coords, np.float64)
            cp, nn = _dp(self._coords), self._coords.shape[0]
        _check(lib.or_precond_build(sys.h, VARIANT[variant], 0 if inner == "amg" else 1, _dp(d),
                                    i.ctypes.data_as(C.POINTER(C.c_int)), cp, nn, C.byref(self.h)))
        self.set_factor_solve(factor_solve)
        if inner == "amg":
            self.set_row_sum(row_sum)

    def set_row_sum(self, mode: str) -> None:
        """'ordered' (the reference's spmv / spmv_transpose order) or 'strided' (extension:
        32 lane-strided partials + xor tree on A_l, l >= 1, and on R_l = P_l^T)."""
        assert mode in ("ordered", "strided"), mode
        _check(lib.or_precond_set_row_sum(self.h, 1 if mode == "strided" else 0))
        self.row_sum = mode

    def set_factor_solve(self, mode: str) -> None:
        """'sweep' (SparseFactor::solve), 'inverse' (explicit block inverse) or 'panel'
        (block-bidiagonal panels; factors without row interchanges)."""
        codes = {"sweep": 0, "inverse": 1, "panel": 2}
        assert mode in codes, mode
        _check(lib.or_precond_set_factor_solve(self.h, codes[mode]))
        self.factor_solve = mode

    def factor_pivots(self) -> bool:
        return bool(lib.or_precond_factor_pivots(self.h))

    def __del__(self):
        if getattr(self, "h", None) and lib is not None:
            lib.or_precond_destroy(self.h)
            self.h = None

    def apply(self, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float64)
        y = np.zeros(self.sys.n)
        _check(lib.or_precond_apply(self.h, _dp(x), _dp(y)))
        return y

    def inner_calls(self, reset=False) -> int:
        return int(lib.or_precond_inner_calls(self.h, int(reset)))

    def n_levels(self) -> int:
        return lib.or_amg_levels(self.h)

    def level_matrix(self, level: int, which: int) -> tuple:
        return csr_from(lib.or_amg_level_matrix(self.h, level, which))

    def level_lambda(self, level: int) -> float:
        """Chebyshev lambda_max estimate of the level (0.0 for other smoothers)."""
        return float(lib.or_amg_level_lambda(self.h, level))

    def level_diag(self, level: int) -> np.ndarray:
        n = self.level_matrix(level, 0)[0]
        out = np.zeros(n)
        lib.or_amg_level_diag(self.h, level, _dp(out))
        return out

    def level_aggregates(self, level: int) -> np.ndarray:
        n = self.level_matrix(level - 1, 0)[0]
        out = np.zeros(n, np.int32)
        lib.or_amg_level_aggregates(self.h, level, out.ctypes.data_as(C.POINTER(C.c_int)))
        return out

    def matrix(self, which: int) -> tuple:
        return csr_from(lib.or_precond_matrix(self.h, which))

    def hblocks(self) -> np.ndarray:
        out = np.zeros(9 * self.sys.n_p)
        lib.or_precond_hblocks(self.h, _dp(out))
        return out

    def vec(self) -> np.ndarray:
        out = np.zeros(self.sys.n_p)
        lib.or_precond_vec(self.h, 0, _dp(out))
        return out

    def level_colors(self, level: int) -> tuple:
        """mcgs (extension): (rows grouped by colour, colour offsets) of a level."""
        nc = lib.or_amg_level_colors(self.h, level, None, None)
        n = self.level_matrix(level, 0)[0]
        rows, off = np.zeros(n, np.int32), np.zeros(nc + 1, np.int32)
        lib.or_amg_level_colors(self.h, level, rows.ctypes.data_as(C.POINTER(C.c_int)),
                                off.ctypes.data_as(C.POINTER(C.c_int)))
        return rows, off

    def amg_apply(self, r: np.ndarray) -> np.ndarray:
        r = np.ascontiguousarray(r, np.float64)
        x = np.zeros(r.size)
        _check(lib.or_amg_apply(self.h, _dp(r), _dp(x)))
        return x


def oracle_gmres(sys: OracleSystem, pc, b, tol=1e-10, restart=50, max_iter=500, scaled=True):
    b = np.ascontiguousarray(b, np.float64)
    x = np.zeros(sys.n)
    st = np.zeros(5, np.int32)
    hist = np.zeros(max_iter + 1)
    secs = np.zeros(1)
    _check(lib.or_gmres(sys.h, pc.h if pc is not None else None, _dp(b), tol, restart, max_iter, int(scaled), _dp(x),
                        st.ctypes.data_as(C.POINTER(C.c_int)), _dp(hist), hist.size, _dp(secs)))
    return x, dict(iterations=int(st[0]), converged=bool(st[1]), breakdown=bool(st[2]), restarts=int(st[3]),
                   precond_applies=int(st[4]), history=hist[: st[0]].copy(), seconds=float(secs[0]))


def mm_read(path: str) -> tuple:
    """read_matrix_market (mmio.cpp:15-48) restated: (rows, cols, rp, ci, v)."""
    h = C.c_void_p()
    _check(lib.or_mm_read(str(path).encode(), C.byref(h)))
    try:
        return csr_from(h)
    finally:
        lib.or_csr_destroy(h)


def mm_write(path: str, rows: int, cols: int, rp, ci, v) -> None:
    rp = np.ascontiguousarray(rp, np.int64)
    ci = np.ascontiguousarray(ci, np.int32)
    v = np.ascontiguousarray(v, np.float64)
    _check(lib.or_mm_write(str(path).encode(), rows, cols, rp.ctypes.data_as(C.POINTER(C.c_int64)),
                           ci.ctypes.data_as(C.POINTER(C.c_int)), _dp(v)))
