"""Device CRC32 (rk_dev_crc32: per-range CTA, slice CRCs combined over GF(2)) against
zlib's CRC-32, and rk_write_records (payload CRCs on the GPU) byte-identical to the
host writer and to the unmodified reference's write_block_record."""
import ctypes as C
import os
import zlib

import numpy as np
import pytest

import paper_2009_09767_b200 as rk
from paper_2009_09767_b200 import configs
from paper_2009_09767_b200 import ranky as R

pytestmark = pytest.mark.gpu


def test_device_crc32_matches_zlib():
    import torch
    rng = np.random.default_rng(5)
    host = rng.integers(0, 256, 3 << 20, dtype=np.uint8)
    dev = torch.from_numpy(host).cuda()
    ranges = [(0, 0), (1, 1), (3, 7), (8, 8), (5, 255), (0, 256), (17, 257), (100, 4099), (7, (1 << 20) + 5),
              (0, 3 << 20)]
    off = np.array([r[0] for r in ranges], dtype=np.uint64)
    ln = np.array([r[1] for r in ranges], dtype=np.uint64)
    crc = np.zeros(len(ranges), dtype=np.uint32)
    R._check(R.lib().rk_dev_crc32(rk.ranky.default_context().handle, C.c_void_p(dev.data_ptr()),
                                  off.ctypes.data_as(C.POINTER(C.c_uint64)), ln.ctypes.data_as(C.POINTER(C.c_uint64)),
                                  len(ranges), crc.ctypes.data_as(C.POINTER(C.c_uint32))))
    for (o, n), c in zip(ranges, crc):
        assert int(c) == zlib.crc32(host[o:o + n].tobytes()), (o, n)


def test_write_records_byte_identical(tmp_path, ref):
    cfg = configs.CONFIGS["c1"]
    a = cfg.generate()
    res = rk.run_pipeline(a, cfg.blocks, cfg.method, 0, cfg.seed, 1, want_records=True)
    R.write_records(res.records, str(tmp_path / "gpu_"))
    for rec in res.records:
        host_path = tmp_path / f"host_{rec.block_index}.rnky"
        R.write_block_record(rec, host_path)
        got = open(tmp_path / f"gpu_{rec.block_index}.rnky", "rb").read()
        assert got == open(host_path, "rb").read()
        if ref.kind == "reference":
            ref.write_block_record(rec.block_index, rec.payload.reshape(rec.rows, rec.kept), tmp_path / "ref.rnky")
            assert got == open(tmp_path / "ref.rnky", "rb").read()
        assert R.read_block_record(tmp_path / f"gpu_{rec.block_index}.rnky") == rec
