"""Validation ingest (formats.py over the native gs_jsonl_* reader): the
reference's JSONL semantics pinned by tests/golden/ingest.json (produced by
gearserve.formats.load_validation), and the columnar container round trip.
Host code only: no GPU needed."""

import json
import math

import numpy as np
import pytest

from conftest import GOLDEN

from paper_2406_14424_b200 import formats
from paper_2406_14424_b200.types import ModelOutput, ValidationRecord, ValidationSet


def _expected():
    return json.loads((GOLDEN / "ingest.json").read_text())


def _same_float(a: float, b: float) -> bool:
    return (math.isnan(a) and math.isnan(b)) or a == b


def test_edge_cases_match_reference_reader():
    want = _expected()["ok"]
    got = formats.load_validation(GOLDEN / "ingest_ok.jsonl", n_threads=3)
    assert len(got) == len(want)
    by_id = {r.sample_id: r for r in got.records}
    for rec in want:
        r = by_id[rec["sample_id"]]
        assert set(r.outputs) == set(rec["models"])
        for mid, out in rec["models"].items():
            assert r.outputs[mid].correct == out["correct"]
            ref = [float(x) for x in out["scores"]]
            assert len(r.outputs[mid].scores) == len(ref)
            assert all(_same_float(a, b) for a, b in zip(r.outputs[mid].scores, ref))


@pytest.mark.parametrize("name", ["missing_correct", "empty_scores", "not_json", "duplicate_id",
                                  "model_mismatch", "negative_id", "bad_score"])
def test_malformed_files_raise_like_the_reference(name):
    want = _expected()["bad"][name]
    path = GOLDEN / f"ingest_bad_{name}.jsonl"
    with pytest.raises(ValueError) as e:
        formats.load_validation(path)
    assert str(path) in str(e.value)
    if want["line"] is not None:
        assert f"line {want['line']}:" in str(e.value)


def test_arrays_view_of_the_same_file():
    arr = formats.load_validation_arrays(GOLDEN / "ingest_ok.jsonl")
    vs = formats.load_validation(GOLDEN / "ingest_ok.jsonl")
    assert len(arr) == len(vs)
    ids = list(arr.model_ids_ordered)
    assert ids == ["a", "b"]  # first record's key order
    for i, r in enumerate(vs.records):
        assert int(arr.sample_id[i]) == r.sample_id
        for j, m in enumerate(ids):
            k = len(r.outputs[m].scores)
            rl = arr.row_len.get(m) if arr.row_len else None
            assert (int(rl[i]) if rl is not None else arr.scores[m].shape[1]) == k
            row = arr.scores[m][i, :k]
            assert all(_same_float(a, b) for a, b in zip(row, r.outputs[m].scores))
            assert int(arr.correct[i, j]) == int(r.outputs[m].correct)


def _random_set(rng, n, ids, ragged):
    recs = []
    for i in range(n):
        outs = {}
        for m in ids:
            k = int(rng.integers(1, 5)) if ragged else 2
            outs[m] = ModelOutput(scores=tuple(float(x) for x in rng.random(k)),
                                  correct=bool(rng.random() < 0.6))
        recs.append(ValidationRecord(sample_id=int(3 * i + 1), outputs=outs))
    return ValidationSet(recs)


@pytest.mark.parametrize("ragged,threads", [(False, 1), (True, 4), (True, 64)])
def test_jsonl_round_trip_many_threads(tmp_path, ragged, threads):
    rng = np.random.default_rng(5)
    vs = _random_set(rng, 2500, ["tiny", "mini", "base"], ragged)
    path = tmp_path / "v.jsonl"
    formats.save_validation(vs, path)
    back = formats.load_validation(path, n_threads=threads)
    assert back == vs


def test_columnar_round_trip(tmp_path):
    rng = np.random.default_rng(6)
    vs = _random_set(rng, 1000, ["m0", "m1"], ragged=True)
    p = tmp_path / "v.gsvc"
    formats.save_validation_columnar(vs, p)
    arr = formats.load_validation_columnar(p)
    ids, sid, scores, row_len, corr = formats._columns(vs)
    assert list(arr.model_ids_ordered) == ids
    assert np.array_equal(arr.sample_id, sid)
    assert np.array_equal(np.asarray(arr.correct), corr)
    for j, m in enumerate(ids):
        assert np.array_equal(arr.scores[m], scores[j])
        rl = (arr.row_len or {}).get(m)
        assert np.array_equal(rl if rl is not None else np.full(len(vs), scores[j].shape[1]),
                              row_len[:, j])
    # the columnar file of a columnar set is the same file again
    p2 = tmp_path / "v2.gsvc"
    formats.save_validation_columnar(arr, p2)
    assert p.read_bytes() == p2.read_bytes()


def test_columnar_rejects_foreign_files(tmp_path):
    p = tmp_path / "x.gsvc"
    p.write_bytes(b"not a container at all")
    with pytest.raises(ValueError):
        formats.load_validation_columnar(p)


def test_number_tokens_and_int_sample_ids(tmp_path):
    """json.loads's number grammar (no hex, no bare inf / nan, no leading '+';
    NaN / Infinity literals accepted) and int() of the sample id: integer
    tokens exactly (past 2^53), floats truncated, decimal strings, bools."""
    def rec(sid, score="0.5"):
        return f'{{"sample_id": {sid}, "models": {{"a": {{"scores": [{score}], "correct": true}}}}}}'

    ok = tmp_path / "ok.jsonl"
    ok.write_text("\n".join([rec(9007199254740993), rec("3.9"), rec('" 12 "'), rec("true"),
                             rec(7, "NaN"), rec(8, "-Infinity"), rec(9, "1e-3")]) + "\n")
    vs = formats.load_validation(ok)
    assert [r.sample_id for r in vs.records] == [9007199254740993, 3, 12, 1, 7, 8, 9]
    assert math.isnan(vs.records[4].outputs["a"].scores[0])
    assert vs.records[5].outputs["a"].scores[0] == -math.inf
    for bad in (rec(1, "0x1p3"), rec(1, "inf"), rec(1, "nan"), rec(1, "+1.0"), rec("NaN"), rec('"1.5"'),
                rec(1, "1."), rec(1, ".5")):
        path = tmp_path / "bad.jsonl"
        path.write_text(bad + "\n")
        with pytest.raises(ValueError):
            formats.load_validation(path)
