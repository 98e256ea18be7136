"""Front-ends either side of the hot path: PGM P5
I/O, synthetic generators, counter reports, the scikit-learn estimator and
the CLI -- pinned to fixtures recorded from the reference
(tests/golden/make_frontend_golden.py -> tests/golden/frontend.json)."""

import contextlib
import hashlib
import io
import json
import os

import numpy as np
import pytest

import paper_1105_3829_b200 as mtb
from paper_1105_3829_b200 import cli
from paper_1105_3829_b200.counters import OpCounters, counters_report

G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "frontend.json")))


def _sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


@pytest.mark.parametrize("case", G["gen"], ids=lambda c: f"{c['kind']}-{c['depth']}-{c['seed']}")
def test_gen_image_matches_reference(case):
    params = {k: tuple(v) if isinstance(v, list) else v for k, v in case["params"].items()}
    im = mtb.gen_image(case["kind"], 37, 23, case["depth"], case["seed"], **params)
    assert str(im.pixels.dtype) == case["dtype"]
    assert im.pixels.ravel()[:6].tolist() == case["first"]
    assert _sha(im.pixels.tobytes()) == case["sha"]


def test_gen_image_errors_match_reference():
    for e in G["gen_errors"]:
        with pytest.raises(ValueError) as ei:
            if e["args"] is None:
                mtb.gen_image("constant", 4, 4, 8, 0, bogus=1)
            else:
                mtb.gen_image(*e["args"])
        assert str(ei.value) == e["msg"]


@pytest.mark.parametrize("case", G["pgm"], ids=lambda c: f"{c['kind']}-{c['depth']}")
def test_write_pgm_bytes_match_reference(case, tmp_path):
    im = mtb.gen_image(case["kind"], 19, 11, case["depth"], case["seed"])
    path = tmp_path / "x.pgm"
    mtb.write_pgm(im, path)
    assert _sha(path.read_bytes()) == case["sha"]
    assert mtb.read_pgm(path) == im  # round trip


@pytest.mark.parametrize("case", G["pgm_errors"], ids=lambda c: c["case"])
def test_read_pgm_cases_match_reference(case, tmp_path):
    path = tmp_path / "x.pgm"
    path.write_bytes(bytes.fromhex(case["data"]))
    if case["ok"]:
        im = mtb.read_pgm(path)
        assert im.bit_depth == case["bits"] and im.pixels.tolist() == case["pixels"]
    else:
        with pytest.raises(mtb.PgmFormatError) as ei:
            mtb.read_pgm(path)
        assert str(ei.value) == case["msg"]
        assert isinstance(ei.value, ValueError)


def test_counters_report_matches_reference():
    r = G["report"]
    rows = [("tree-uniform-n11", OpCounters.from_tally(r["tally"], r["pixels"])), ("b", OpCounters(pixels=5))]
    assert counters_report(rows, "human") == r["human"]
    assert counters_report(rows, "csv") == r["csv"]
    with pytest.raises(ValueError):
        counters_report(rows, "xml")


@pytest.mark.parametrize("case", G["estimator_errors"], ids=lambda c: str(c["params"]))
def test_estimator_validation_matches_reference(case):
    img = np.arange(64, dtype=np.uint8).reshape(8, 8)
    est = mtb.MedianFilter2D(**case["params"])
    if case["msg"] is None:
        est.fit(img)
    else:
        with pytest.raises(ValueError) as ei:
            est.fit(img)
        assert str(ei.value) == case["msg"]


def test_estimator_is_a_sklearn_transformer():
    from sklearn.base import clone
    from sklearn.exceptions import NotFittedError

    est = mtb.MedianFilter2D(window=5, rank=3, mode="adaptive")
    assert clone(est).get_params() == est.get_params()
    with pytest.raises(NotFittedError):
        est.transform(np.zeros((8, 8), np.uint8))
    est.fit(np.zeros((8, 8), np.uint16))
    with pytest.raises(ValueError, match="fitted on 16-bit"):
        est.transform(np.zeros((8, 8), np.uint8))


def _run_cli(argv):
    out, err = io.StringIO(), io.StringIO()
    with contextlib.redirect_stdout(out), contextlib.redirect_stderr(err):
        code = cli.main(argv)
    return code, out.getvalue(), err.getvalue()


def test_cli_errors_match_reference():
    for c in G["cli"]:
        if c["code"] != 2:
            continue
        assert _run_cli(c["argv"]) == (c["code"], c["stdout"], c["stderr"])


# ---------------------------------------------------------------- GPU side

@pytest.mark.gpu
def test_cli_compare_lines_match_reference():
    for c in G["cli"]:
        if c["argv"][0] != "compare":
            continue
        assert _run_cli(c["argv"]) == (c["code"], c["stdout"], c["stderr"])


@pytest.mark.gpu
def test_cli_filter_pgm_matches_reference(tmp_path):
    path = tmp_path / "o.pgm"
    code, out, _ = _run_cli(G["cli_filter_pgm"]["argv"] + ["-o", str(path)])
    assert code == 0 and "tree-uniform-n5" in out
    assert _sha(path.read_bytes()) == G["cli_filter_pgm"]["sha"]


@pytest.mark.gpu
def test_cli_bench_csv(tmp_path):
    csv = tmp_path / "c.csv"
    code, _, err = _run_cli(["bench", "--gen", "normal_noise", "--width", "64", "--height", "48",
                             "-n", "3", "--windows", "3,5", "--oracle", "huang", "--counters", str(csv)])
    assert code == 0 and "tree-uniform-n5" in err
    lines = csv.read_text().splitlines()
    assert lines[0] == mtb.CSV_HEADER and len(lines) == 5
    assert lines[3] == f"huang-n3,0,0,{48 * (9 + 63 * 6)},0,0,0,{48 * (9 + 63 * 6)},0,0.000000,{64 * 48}"


@pytest.mark.gpu
def test_estimator_transform_matches_oracle():
    from oracle import oracle as O

    rng = np.random.default_rng(3)
    img = rng.integers(0, 256, (60, 70)).astype(np.uint8)
    for params in ({"window": 7}, {"window": 9, "rank": 5}, {"window": 5, "percentile": 0.9},
                   {"window": 11, "max_error": 8}):
        est = mtb.MedianFilter2D(**params).fit(img)
        n = params["window"]
        rank = params.get("rank")
        if "percentile" in params:
            rank = int(np.ceil(params["percentile"] * n * n))
        got = est.transform(img)
        assert np.array_equal(got, O.iot_filter(img, n, rank=rank, max_error=params.get("max_error", 1)))
        assert est.counters_.pixels == img.size
    img16 = mtb.gen_image("two_mode", 50, 40, 16, 1).pixels
    est = mtb.MedianFilter2D(window=7, mode="adaptive").fit(img16)
    assert np.array_equal(est.transform(img16), O.iot_filter(img16, 7))


@pytest.mark.gpu
@pytest.mark.parametrize("bits", [8, 16])
def test_bruteforce_oracle_matches_c_oracle(bits):
    from oracle import oracle as O

    rng = np.random.default_rng(bits)
    px = rng.integers(0, 1 << bits, (45, 52)).astype(np.uint8 if bits == 8 else np.uint16)
    for n, rank in ((3, None), (7, 1), (9, 81), (11, 30)):
        ref = O.iot_filter(px, n, rank=rank)
        got = mtb.oracle_median_filter(px, n, rank).pixels
        assert np.array_equal(got, ref)
        out, adds = mtb.huang_filter(px, n, rank)
        assert np.array_equal(out.pixels, ref) and adds == 45 * (n * n + 51 * 2 * n)


def test_window_engine_host_checks():
    img = mtb.gen_image("normal_noise", 9, 7, 8, 1)
    with pytest.raises(ValueError, match="topology is 16-bit, image is 8-bit"):
        mtb.WindowEngine(img, 3, mtb.uniform_topology(16))
    with pytest.raises(ValueError):
        mtb.WindowEngine(img, 4, mtb.uniform_topology(8))


def test_descent_intervals_agree_with_recorded_steps():
    """(value, bound) is a function of the exact value: every recorded step
    of the reference must be descent_intervals() of some value (CPU check
    of the interval tables themselves)."""
    for c in G["window_engine"]:
        im = mtb.gen_image(c["kind"], 9, 7, c["depth"], c["seed"])
        topo = mtb.resolve_topology(im, c["n"], c["mode"])
        lo, width = mtb.descent_intervals(topo, c["max_error"])
        pairs = set(zip(lo.tolist(), width.tolist()))
        assert all(tuple(s) in pairs for s in c["steps"])


@pytest.mark.gpu
def test_window_engine_steps_match_reference():
    for c in G["window_engine"]:
        im = mtb.gen_image(c["kind"], 9, 7, c["depth"], c["seed"])
        topo = mtb.resolve_topology(im, c["n"], c["mode"])
        eng = mtb.WindowEngine(im, c["n"], topo, rank=c["rank"], max_error=c["max_error"])
        assert eng.position == (0, 0)
        steps = [list(s) for s in eng]
        assert steps == c["steps"], (c["mode"], c["max_error"])
        assert eng.position == (0, 7) and eng.counters.pixels == 63
        with pytest.raises(StopIteration):
            eng.step()
        with pytest.raises(RuntimeError, match="fresh engine"):
            eng.run()
        eng2 = mtb.WindowEngine(im, c["n"], topo, rank=c["rank"], max_error=c["max_error"])
        assert eng2.run().tolist() == c["run"]
