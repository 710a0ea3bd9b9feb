"""Matrix Market I/O and the schema-v1 run record against
files and records produced by the unmodified reference
(tests/golden/make_golden.py gen_io): the reader reproduces the reference
reader's double-double planes bit for bit, the writer reproduces the
reference writer's text byte for byte, and records validate both ways."""
import json
import os

import numpy as np
import pytest

from paper_2203_10879_b200 import RefineConfig, RefineReport, RefineStatus, VerifyResiduals
from paper_2203_10879_b200 import matrix_market as mm
from paper_2203_10879_b200 import run_record as rr

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def io_ref():
    return np.load(os.path.join(HERE, "io_ref.npz"))


@pytest.mark.parametrize("tag", ["dd_complex", "f64_real", "coord_sym"])
def test_reader_matches_reference_reader(io_ref, tag):
    got = mm.read_matrix_market(os.path.join(HERE, "mm_%s.mtx" % tag))
    for cell, arr in zip(("rh", "rl", "ih", "il"), got):
        want = io_ref["%s_%s" % (tag, cell)]
        assert arr.shape == want.shape and np.array_equal(arr, want), (tag, cell)


def test_writer_matches_reference_writer_bytes(io_ref, tmp_path):
    src = tuple(io_ref["src_%s" % c] for c in ("rh", "rl", "ih", "il"))
    path = tmp_path / "w.mtx"
    mm.write_matrix_market(str(path), src, comment="reference writer, dd")
    assert path.read_text() == open(os.path.join(HERE, "mm_dd_complex.mtx")).read()
    # and it round-trips bit for bit
    back = mm.read_matrix_market(str(path))
    for a, b in zip(back, src):
        assert np.array_equal(a + 0.0, b + 0.0) or np.array_equal(a, b)


def test_binary64_round_trip_and_metadata(tmp_path):
    rng = np.random.default_rng(1)
    x = rng.standard_normal((6, 3)) + 1j * rng.standard_normal((6, 3))
    p = tmp_path / "c.mtx"
    mm.write_matrix_market(str(p), x)
    back = mm.read_matrix_market(str(p))
    assert np.array_equal(back[0] + back[1] + 1j * (back[2] + back[3]), x)
    assert mm.header_metadata(str(p)) == ("array", "complex", "general", (6, 3))
    assert mm.header_metadata(os.path.join(HERE, "mm_coord_sym.mtx"))[3] == (4, 4, 5)


@pytest.mark.parametrize("text", [
    "%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n",           # too few values
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n",    # index out of range
    "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1\n1 1 2\n",  # duplicate
    "%%MatrixMarket matrix coordinate real symmetric\n2 2 1\n1 2 1.0\n",  # upper entry
    "%%MatrixMarket vector array real general\n2\n1\n2\n",                 # object
    "%%MatrixMarket matrix array real general\n2 2\n1\n2\nx\n4\n",        # bad value
])
def test_reader_rejects_malformed(tmp_path, text):
    p = tmp_path / "bad.mtx"
    p.write_text(text)
    with pytest.raises(mm.MatrixMarketError):
        mm.read_matrix_market(str(p))


def test_run_record_schema_v1():
    ref = json.load(open(os.path.join(HERE, "run_record_ref.json")))
    assert rr.validate_run_record(ref) is ref
    rep = RefineReport(iterations=ref["report"]["iterations"],
                       residual_history=[tuple(r) for r in ref["report"]["residual_history"]],
                       hp_matmul_count=ref["report"]["hp_matmul_count"], clipped_total=0,
                       status=RefineStatus(ref["report"]["status"]), wall_time=ref["report"]["wall_time"],
                       skip_fired=ref["report"]["skip_fired"], detail=ref["report"]["detail"])
    res = VerifyResiduals(*(ref["residuals"][k] for k in rr.RESIDUAL_KEYS))
    spec = rr.make_spec("randn", 8, seed=1)
    ours = rr.build_run_record(spec, RefineConfig(seed=1), rep, res)
    assert json.loads(rr.dumps(ours)) == ref
    bad = dict(ours)
    bad["report"] = dict(ours["report"], residual_history=ours["report"]["residual_history"][:-1])
    with pytest.raises(ValueError):
        rr.validate_run_record(bad)
    with pytest.raises(ValueError):
        rr.validate_run_record(dict(ours, extra=1))
    nonfinite = dict(ours, residuals=rr.residuals_to_dict(VerifyResiduals(float("nan"), 1.0, float("inf"))))
    assert nonfinite["residuals"]["ortho_residual"] is None and nonfinite["residuals"]["similarity_residual"] is None
