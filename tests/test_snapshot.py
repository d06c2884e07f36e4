"""Snapshot bundle I/O (snapshot.cpp:28-104, mmio.cpp:15-76): the product's
parallel Matrix Market reader/writer and manifest handling against the oracle's
sequential restatement, the round trip, and the reference's error cases."""
import filecmp
import json
import os

import numpy as np
import pytest

import oracle_lib as O
from paper_2112_12397_b200 import api
from test_abi_cpu import small_workload

BLOCKS = ("A", "C1", "Q1", "C2", "H", "Q2", "T", "F_u")


def same(m: api.CsrMatrix, t: tuple) -> bool:
    r, c, rp, ci, v = t
    return (m.n_rows, m.n_cols) == (r, c) and np.array_equal(m.row_offsets, rp) and \
        np.array_equal(m.col_indices, ci) and np.array_equal(m.values.view(np.uint64), v.view(np.uint64))


def test_round_trip_is_bitwise_and_matches_the_oracle_reader(tmp_path):
    W = api.Workload(spec=dict(cells=(6, 6, 5), fractures=[(0, 0.5, 0.0, 1.0, 0.0, 1.0)], frac_stick=0.5,
                               frac_slip=0.3, E_sigma_ln=0.5, aperture_sigma_ln=0.3), seed=5)
    J = W.system()
    region, dt = W.region()
    assert len(region) == J.n_p and set(region) <= set("slo") and dt == 0.5
    d = tmp_path / "snap"
    W.save_snapshot(str(d))
    man = json.load(open(d / "manifest.json"))
    assert (man["n_u"], man["n_t"], man["n_p"], man["dt"], man["region"]) == (J.n_u, J.n_t, J.n_p, 0.5, region)
    assert man["blocks"] == {b: f"{b}.mtx" for b in BLOCKS} and man["coords"] == "coords.txt"
    W2 = api.Workload.from_snapshot(str(d))
    J2 = W2.system()
    assert W2.region() == (region, dt)
    assert np.array_equal(J2.node_coords, J.node_coords)
    for b in BLOCKS:
        m, m2 = getattr(J, b), getattr(J2, b)
        assert same(m2, (m.n_rows, m.n_cols, m.row_offsets, m.col_indices, m.values)), b
        assert same(m2, O.mm_read(str(d / f"{b}.mtx"))), b  # oracle reader, same file
        # the writer is byte-identical to the oracle's (the reference's printf formats)
        O.mm_write(str(tmp_path / f"ref_{b}.mtx"), m.n_rows, m.n_cols, m.row_offsets, m.col_indices, m.values)
        assert filecmp.cmp(d / f"{b}.mtx", tmp_path / f"ref_{b}.mtx", shallow=False), b
    info = W2.info()
    assert (info["stick"], info["slip"], info["open"]) == (region.count("s"), region.count("l"), region.count("o"))


def _tiny_bundle(d, A_text: str, region="s", dt=0.25, extra=None):
    """n_u = 3, n_p = 1 system whose A.mtx is hand-written."""
    d.mkdir(parents=True, exist_ok=True)
    (d / "A.mtx").write_text(A_text)
    eye = lambda r, c: O.mm_write(str(d / f"{nm}.mtx"), r, c, np.arange(min(r, c) + 1).tolist() +  # noqa: E731
                                  [min(r, c)] * (r - min(r, c)), list(range(min(r, c))), [1.0] * min(r, c))
    for nm, (r, c) in {"C1": (3, 3), "Q1": (3, 1), "C2": (3, 3), "H": (3, 3), "Q2": (1, 3), "T": (1, 1),
                       "F_u": (1, 3)}.items():
        eye(r, c)
    man = {"n_u": 3, "n_t": 3, "n_p": 1, "dt": dt, "region": region, "blocks": {b: f"{b}.mtx" for b in BLOCKS}}
    man.update(extra or {})
    (d / "manifest.json").write_text(json.dumps(man, indent=2))


def test_reader_semantics_duplicates_order_comments(tmp_path):
    text = ("%%MatrixMarket matrix coordinate real general\n% a comment\n\n%another\n3 3 7\n"
            "3 1 +2.5\n1 2 1e-3\n1 2 -4\n2 2 0.1\n1 1 7\n3 1 1.25e0\n2 3 -0.0\n")
    d = tmp_path / "b"
    _tiny_bundle(d, text)
    J = api.Workload.from_snapshot(str(d)).system()
    ref = O.mm_read(str(d / "A.mtx"))
    assert same(J.A, ref)
    # stable (row, col) order, duplicates summed from 0.0 in file order
    assert J.A.col_indices.tolist() == [0, 1, 1, 2, 0]
    assert J.A.values.tolist() == [7.0, 0.0 + 1e-3 + -4.0, 0.1, -0.0 + 0.0, 0.0 + 2.5 + 1.25]
    assert api.Workload.from_snapshot(str(d)).region() == ("s", 0.25)


def test_parallel_reader_on_a_large_block(tmp_path):
    J = api.Workload(1, 42).system()  # A: 2,074,086 entries, parsed in many chunks
    d = tmp_path / "c1"
    api.export_snapshot(str(d), J, "s" * J.n_p, 0.5)
    J2 = api.Workload.from_snapshot(str(d)).system()
    for b in BLOCKS:
        m = getattr(J, b)
        assert same(getattr(J2, b), (m.n_rows, m.n_cols, m.row_offsets, m.col_indices, m.values)), b
    assert same(J2.A, O.mm_read(str(d / "A.mtx")))


@pytest.mark.parametrize("case,msg", [
    ("header", "unsupported MatrixMarket header"),
    ("symmetric", "only real general coordinate matrices supported"),
    ("size", "bad size line"),
    ("range", "entry out of range"),
    ("truncated", "truncated matrix data"),
    ("badtoken", "truncated matrix data"),
    ("region_label", "bad region label"),
    ("region_len", "region string length mismatch"),
    ("nt", "n_t == 3\\*n_p"),
    ("no_manifest", "missing manifest.json"),
    ("missing_key", "manifest has no \"dt\""),
    ("coords_len", "coords length mismatch"),
    ("not_json", "not valid JSON"),
])
def test_import_errors_follow_the_reference(tmp_path, case, msg):
    good = "%%MatrixMarket matrix coordinate real general\n3 3 3\n1 1 1\n2 2 1\n3 3 1\n"
    d = tmp_path / case
    A = {"header": "%%MatrixMarket matrix array real general\n3 3\n",
         "symmetric": "%%MatrixMarket matrix coordinate real symmetric\n3 3 0\n",
         "size": "%%MatrixMarket matrix coordinate real general\n3 x 3\n",
         "range": "%%MatrixMarket matrix coordinate real general\n3 3 2\n1 1 1\n4 1 1\n",
         "truncated": "%%MatrixMarket matrix coordinate real general\n3 3 3\n1 1 1\n2 2\n",
         "badtoken": "%%MatrixMarket matrix coordinate real general\n3 3 2\n1 1 abc\n9 9 9\n"}.get(case, good)
    extra = {"region_label": {"region": "x"}, "region_len": {"region": "ss"}, "nt": {"n_t": 4},
             "coords_len": {"coords": "coords.txt"}}.get(case)
    _tiny_bundle(d, A, extra=extra)
    if case == "coords_len":
        (d / "coords.txt").write_text("0\n1\n")
    if case == "no_manifest":
        os.remove(d / "manifest.json")
    if case == "missing_key":
        m = json.load(open(d / "manifest.json"))
        del m["dt"]
        (d / "manifest.json").write_text(json.dumps(m))
    if case == "not_json":
        (d / "manifest.json").write_text("{\"n_u\": 3,")
    with pytest.raises(ValueError, match=msg):
        api.Workload.from_snapshot(str(d))
    if case in ("header", "symmetric", "size", "range", "truncated", "badtoken"):
        with pytest.raises(ValueError, match=msg):  # the oracle reader agrees on the error
            O.mm_read(str(d / "A.mtx"))


def test_export_rejects_bad_region(tmp_path):
    J = small_workload()
    with pytest.raises(ValueError, match="region labels size mismatch"):
        api.export_snapshot(str(tmp_path / "x"), J, "s", 0.5)


@pytest.mark.gpu
def test_snapshot_solve_equals_generated_system(tmp_path):
    """A bundle written from a generated system solves exactly like the system itself."""
    W = api.Workload(spec=dict(cells=(8, 6, 6), fractures=[(0, 0.5, 0.0, 1.0, 0.0, 1.0)], frac_stick=0.5,
                               frac_slip=0.3, E_sigma_ln=0.5, aperture_sigma_ln=0.3), seed=9)
    W.save_snapshot(str(tmp_path / "s"))
    W2 = api.Workload.from_snapshot(str(tmp_path / "s"))
    res = []
    for w in (W, W2):
        J = w.system(copy=False)
        op = api.BlockSystemOperator(J)
        pc = api.GpuPreconditioner.from_host(op, api.HostPreconditioner.from_workload(w, api.PrecondConfig("tup")))
        x = np.random.default_rng(3).uniform(-1, 1, J.total_dimension())
        b = np.random.default_rng(4).uniform(-1, 1, J.total_dimension())
        sol, st = api.gmres(op, pc, b, tol=1e-10, max_iter=200, restart=50, scaled=True)
        res.append((pc.apply(x), sol, st.iterations))
    assert np.array_equal(res[0][0], res[1][0])
    assert np.array_equal(res[0][1], res[1][1]) and res[0][2] == res[1][2]
