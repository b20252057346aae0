"""Validation-set formats feeding the sweep.

* The reference's JSONL (``formats.load_validation`` / ``save_validation``,
  /root/reference/pkg/src/gearserve/formats.py:75-106): one record per line,
  ``{"sample_id", "models": {"<id>": {"scores": [...], "correct": bool}}}``.
  ``load_validation`` returns the reference's ``ValidationSet``;
  ``load_validation_arrays`` returns a columnar ``ValidationArrays`` (score
  matrices per model, certainty computed on the device by ``gs_certainty``)
  without building a Python object per record.  Both parse with the native
  multi-threaded reader ``gs_jsonl_open/read`` (csrc/gs_ingest.cu), with the
  reference's semantics and its ``ValueError("<path>: line N: ...")`` errors.
* A columnar binary container (``.gsvc``) for repeated sweeps over the same
  set: ``save_validation_columnar`` / ``load_validation_columnar`` (memory
  mapped; score blocks go to the device as they are).

Layout of ``.gsvc``: magic ``b"GSVC0001"``, u64 header length, a JSON
header ``{"n_records", "models": [{"id", "width", "ragged"}]}``, then
64-byte-aligned blocks: sample_id i64 [n], correct u8 [n, M], and per model
scores f64 [n, width] followed by row_len i32 [n] when ragged.
"""

from __future__ import annotations

import ctypes
import json
import os
from pathlib import Path

import numpy as np

from . import _lib
from .types import ModelOutput, ValidationArrays, ValidationRecord, ValidationSet

MAGIC = b"GSVC0001"
_ALIGN = 64


def _fail(path, msg: str) -> None:
    raise ValueError(f"{path}: {msg}")


class _Parsed:
    def __init__(self, ids, sample_id, scores, row_len, correct):
        self.ids = ids                  # model ids, first-record order
        self.sample_id = sample_id      # [n] int64
        self.scores = scores            # list of [n, width_m] f64
        self.row_len = row_len          # [n, M] int32
        self.correct = correct          # [n, M] uint8


def _parse_jsonl(path, n_threads: int | None = None) -> _Parsed:
    lib = _lib.load()
    info = _lib.gs_jsonl_info()
    handle = ctypes.c_void_p()
    threads = int(n_threads or os.cpu_count() or 1)
    rc = lib.gs_jsonl_open(str(path).encode(), threads, ctypes.byref(handle), ctypes.byref(info))
    if rc != _lib.GS_OK:
        msg = info.error.decode(errors="replace")
        if info.err_line:
            _fail(path, f"line {info.err_line}: {msg}")
        _fail(path, msg)
    try:
        n, m_count = int(info.n_records), int(info.n_models)
        ids = [info.model_ids[j].value.decode() for j in range(m_count)]
        widths = [int(info.width[j]) for j in range(m_count)]
        sample_id = np.empty(n, dtype=np.int64)
        line_no = np.empty(n, dtype=np.int64)
        scores = [np.empty((n, w), dtype=np.float64) for w in widths]
        ptrs = (ctypes.c_void_p * m_count)(*[s.ctypes.data for s in scores])
        row_len = np.empty((n, m_count), dtype=np.int32)
        correct = np.empty((n, m_count), dtype=np.uint8)
        _lib.check(lib.gs_jsonl_read(handle, sample_id.ctypes.data, line_no.ctypes.data, ptrs,
                                     row_len.ctypes.data, correct.ctypes.data), "jsonl read")
    finally:
        lib.gs_jsonl_close(handle)
    # cross-record checks of ValidationSet (src/types.py:160-180), by line
    order = np.argsort(sample_id, kind="stable")
    dup = np.flatnonzero(sample_id[order][1:] == sample_id[order][:-1])
    if dup.size:
        i = order[dup[0] + 1]
        _fail(path, f"line {int(line_no[i])}: duplicate sample_id {int(sample_id[i])}")
    return _Parsed(ids, sample_id, scores, row_len, correct)


def load_validation(path, n_threads: int | None = None) -> ValidationSet:
    """The reference's reader (src/formats.py:75-97): a ValidationSet."""
    p = _parse_jsonl(path, n_threads)
    records = []
    for i in range(p.sample_id.size):
        outs = {}
        for j, mid in enumerate(p.ids):
            k = int(p.row_len[i, j])
            outs[mid] = ModelOutput(scores=tuple(float(x) for x in p.scores[j][i, :k]),
                                    correct=bool(p.correct[i, j]))
        records.append(ValidationRecord(sample_id=int(p.sample_id[i]), outputs=outs))
    try:
        return ValidationSet(records)
    except ValueError as e:
        _fail(path, str(e))


def load_validation_arrays(path, n_threads: int | None = None) -> ValidationArrays:
    """The same file as columnar arrays: score matrices per model (row
    lengths when ragged), correct [n, M], sample ids; certainty is computed
    on the device when the sweep asks for it."""
    p = _parse_jsonl(path, n_threads)
    return _arrays(p.ids, p.sample_id, p.scores, p.row_len, p.correct)


def _arrays(ids, sample_id, scores, row_len, correct) -> ValidationArrays:
    sc, rl = {}, {}
    for j, mid in enumerate(ids):
        sc[mid] = scores[j]
        lens = row_len[:, j]
        if lens.size and int(lens.min()) != scores[j].shape[1]:
            rl[mid] = np.ascontiguousarray(lens)
    return ValidationArrays(ids, scores=sc, correct=correct, row_len=rl or None,
                            sample_id=sample_id)


def save_validation(validation: ValidationSet, path) -> None:
    """The reference's writer (src/formats.py:100-106)."""
    with open(path, "w") as f:
        for r in validation.records:
            doc = {"sample_id": r.sample_id,
                   "models": {mid: {"scores": list(out.scores), "correct": out.correct}
                              for mid, out in r.outputs.items()}}
            f.write(json.dumps(doc) + "\n")


def _columns(validation):
    """(ids, sample_id, scores list, row_len [n, M], correct [n, M])."""
    if isinstance(validation, ValidationArrays):
        if validation.scores is None:
            raise ValueError("columnar files hold score rows; this set has certainty only")
        ids = list(validation.model_ids_ordered)
        n = len(validation)
        scores = [np.ascontiguousarray(np.asarray(validation.scores[m], dtype=np.float64))
                  for m in ids]
        rl = validation.row_len or {}
        row_len = np.stack([np.asarray(rl.get(m, np.full(n, s.shape[1])), dtype=np.int32)
                            for m, s in zip(ids, scores)], axis=1)
        sid = (np.asarray(validation.sample_id, dtype=np.int64)
               if validation.sample_id is not None else np.arange(n, dtype=np.int64))
        corr = (np.asarray(validation.correct) != 0).astype(np.uint8)
        return ids, sid, scores, row_len, corr
    ids = list(validation.records[0].outputs)
    n = len(validation)
    row_len = np.array([[len(r.outputs[m].scores) for m in ids] for r in validation.records],
                       dtype=np.int32).reshape(n, len(ids))
    scores = []
    for j, m in enumerate(ids):
        a = np.zeros((n, int(row_len[:, j].max())), dtype=np.float64)
        for i, r in enumerate(validation.records):
            sc = r.outputs[m].scores
            a[i, : len(sc)] = sc
        scores.append(a)
    corr = np.array([[r.outputs[m].correct for m in ids] for r in validation.records],
                    dtype=np.uint8).reshape(n, len(ids))
    sid = np.array([r.sample_id for r in validation.records], dtype=np.int64)
    return ids, sid, scores, row_len, corr


def save_validation_columnar(validation, path) -> None:
    """Write a ValidationSet / ValidationArrays as a .gsvc container."""
    ids, sid, scores, row_len, corr = _columns(validation)
    n = int(sid.size)
    models = [{"id": m, "width": int(s.shape[1]),
               "ragged": bool(int(row_len[:, j].min()) != s.shape[1])}
              for j, (m, s) in enumerate(zip(ids, scores))]
    header = json.dumps({"n_records": n, "models": models}).encode()
    with open(path, "wb") as f:
        f.write(MAGIC)
        f.write(np.uint64(len(header)).tobytes())
        f.write(header)

        def block(arr):
            pad = (-f.tell()) % _ALIGN
            f.write(b"\0" * pad)
            f.write(np.ascontiguousarray(arr).tobytes())

        block(sid)
        block(corr)
        for j, (mdoc, s) in enumerate(zip(models, scores)):
            block(s.astype(np.float64, copy=False))
            if mdoc["ragged"]:
                block(row_len[:, j].astype(np.int32))


def load_validation_columnar(path) -> ValidationArrays:
    """Memory-map a .gsvc container into a ValidationArrays."""
    path = Path(path)
    with open(path, "rb") as f:
        if f.read(8) != MAGIC:
            _fail(path, "not a gearserve columnar validation file")
        hlen = int(np.frombuffer(f.read(8), dtype=np.uint64)[0])
        try:
            header = json.loads(f.read(hlen).decode())
            n = int(header["n_records"])
            models = header["models"]
        except (ValueError, KeyError, TypeError) as e:
            _fail(path, f"bad header: {e}")
        off = 16 + hlen
    mm = np.memmap(path, dtype=np.uint8, mode="r")

    def take(dtype, shape):
        nonlocal off
        off += (-off) % _ALIGN
        count = int(np.prod(shape)) * np.dtype(dtype).itemsize
        if off + count > mm.size:
            _fail(path, "truncated file")
        arr = np.frombuffer(mm, dtype=dtype, count=int(np.prod(shape)), offset=off).reshape(shape)
        off += count
        return arr

    m_count = len(models)
    sid = take(np.int64, (n,))
    corr = take(np.uint8, (n, m_count))
    ids, scores, row_len = [], [], np.empty((n, m_count), dtype=np.int32)
    for j, md in enumerate(models):
        ids.append(str(md["id"]))
        w = int(md["width"])
        scores.append(take(np.float64, (n, w)))
        row_len[:, j] = take(np.int32, (n,)) if md.get("ragged") else w
    return _arrays(ids, sid, scores, row_len, corr)
