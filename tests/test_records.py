"""RNKY block records on the host path (CPU): mirrors proj/tests/harness_test.cpp
record cases, pinned byte-for-byte against a file written by the unmodified
reference (tests/golden/record_ref.rnky, tests/golden/make_record_golden.py) and
against zlib's CRC-32 (the same polynomial and conventions)."""
import os
import zlib

import numpy as np
import pytest

from paper_2009_09767_b200 import ranky as R

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "record_ref.rnky")


def test_crc32_check_value_and_zlib():
    # harness_test.cpp:31-35
    assert R.crc32(b"123456789") == 0xCBF43926
    assert R.crc32(b"") == 0
    rng = np.random.default_rng(0)
    for n in (1, 7, 8, 9, 255, 256, 4099):
        b = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
        assert R.crc32(b) == zlib.crc32(b)


def test_golden_reference_file(tmp_path):
    raw = open(GOLDEN, "rb").read()
    rec = R.read_block_record(GOLDEN)
    assert rec.block_index == 2 and rec.rows == 6 and rec.kept == 6
    # written again by this implementation: the same bytes
    R.write_block_record(rec, tmp_path / "again.rnky")
    assert open(tmp_path / "again.rnky", "rb").read() == raw
    assert raw[:4] == b"RNKY"


def test_round_trip_and_empty(tmp_path):
    # harness_test.cpp:37-69
    rng = np.random.default_rng(1)
    r = R.BlockResultRecord(3, 5, 4, rng.standard_normal((5, 4)))
    R.write_block_record(r, tmp_path / "a.rnky")
    assert R.read_block_record(tmp_path / "a.rnky") == r
    R.write_block_record(R.read_block_record(tmp_path / "a.rnky"), tmp_path / "b.rnky")
    assert open(tmp_path / "a.rnky", "rb").read() == open(tmp_path / "b.rnky", "rb").read()
    e = R.BlockResultRecord(9, 4, 0, np.zeros((4, 0)))
    R.write_block_record(e, tmp_path / "e.rnky")
    back = R.read_block_record(tmp_path / "e.rnky")
    assert back == e and back.payload.size == 0
    with pytest.raises(R.InvalidArgument, match="payload size mismatch"):
        R.write_block_record(R.BlockResultRecord(1, 3, 2, np.zeros(5)), tmp_path / "x.rnky")


def test_corruption_and_malformed(tmp_path):
    # harness_test.cpp:71-126
    path = tmp_path / "c.rnky"
    raw = open(GOLDEN, "rb").read()
    rng = np.random.default_rng(1234)
    pay_begin, pay_bytes = 18, len(raw) - 18 - 4
    for _ in range(100):
        b = bytearray(raw)
        i = pay_begin + int(rng.integers(pay_bytes))
        b[i] ^= 1 << int(rng.integers(8))
        open(path, "wb").write(b)
        with pytest.raises(R.RecordError, match="checksum mismatch"):
            R.read_block_record(path)
    cases = {"bad block record magic": b"X" + raw[1:], "unsupported block record version": raw[:4] + b"\x02" + raw[5:],
             "payload truncated": raw[:-9], "block record truncated": raw[:10]}
    for msg, b in cases.items():
        open(path, "wb").write(b)
        with pytest.raises(R.RecordError, match=msg):
            R.read_block_record(path)
    with pytest.raises(R.RankyRuntimeError, match="cannot open"):
        R.read_block_record(tmp_path / "missing.rnky")


def test_against_live_reference(ref, tmp_path):
    if ref.kind != "reference":
        pytest.skip("reference library not built")
    rng = np.random.default_rng(2)
    pay = rng.standard_normal((7, 3))
    ref.write_block_record(11, pay, tmp_path / "ref.rnky")
    R.write_block_record(R.BlockResultRecord(11, 7, 3, pay), tmp_path / "ours.rnky")
    assert open(tmp_path / "ref.rnky", "rb").read() == open(tmp_path / "ours.rnky", "rb").read()
    idx, back = ref.read_block_record(tmp_path / "ours.rnky")
    assert idx == 11 and np.array_equal(back, pay)
