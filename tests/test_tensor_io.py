"""OURO tensor files (tensor_io.hpp:13-44): the C ABI's
tensor_save / tensor_load against the reference's own write_tensor_* /
read_tensor_* (oracle/_ref): byte-identical files both ways for f64, i8 and u4
(odd element counts: the trailing high nibble stays 0), the packed-u4 path that
writes a K1 operand's device bytes unchanged, and the reference's error classes."""
import os

import numpy as np
import pytest

import paper_2503_10959_b200 as ob

SHAPES = [(3, 5), (2, 4), (7,), (1, 1, 9)]


def _codes(shape, lo, hi, seed):
    return np.random.default_rng(seed).integers(lo, hi + 1, size=shape, dtype=np.int64).astype(np.int8)


@pytest.mark.parametrize("dtype", [ob.DTYPE_F64, ob.DTYPE_I8, ob.DTYPE_U4])
@pytest.mark.parametrize("shape", SHAPES)
def test_files_byte_identical_to_reference(ref_checker, tmp_path, dtype, shape):
    if dtype == ob.DTYPE_F64:
        data = np.random.default_rng(1).standard_normal(shape)
    else:
        data = _codes(shape, -8 if dtype == ob.DTYPE_U4 else -128, 7 if dtype == ob.DTYPE_U4 else 127, 2)
    ours, ref = tmp_path / "ours.ouro", tmp_path / "ref.ouro"
    ob.tensor_save(ours, data, dtype)
    ref_checker.ref_write_tensor(ref, dtype, data)
    assert ours.read_bytes() == ref.read_bytes()
    assert ob.tensor_info(ref) == (dtype, tuple(shape))
    back = ob.tensor_load(ref)
    assert back.shape == tuple(shape) and np.array_equal(back, data)
    if dtype != ob.DTYPE_F64:  # the reference reads ours
        assert np.array_equal(ref_checker.ref_read_tensor_codes(ours, dtype, data.size), data.ravel())


def test_packed_u4_payload_is_the_device_layout(ref_checker, tmp_path):
    """A [rows][E] code matrix nibble-packed per row (low nibble = even column,
    the K1 operand layout with OURO_B200_CODES_PACKED_I4) is the u4 payload."""
    codes = _codes((6, 32), -7, 7, 3)
    u = codes.astype(np.uint8) & 0x0F
    packed = (u[:, 0::2] | (u[:, 1::2] << 4)).astype(np.uint8)
    ob.tensor_save(tmp_path / "p.ouro", packed, ob.DTYPE_U4, packed=True, shape=codes.shape)
    ref_checker.ref_write_tensor(tmp_path / "r.ouro", ob.DTYPE_U4, codes)
    assert (tmp_path / "p.ouro").read_bytes() == (tmp_path / "r.ouro").read_bytes()
    assert np.array_equal(ob.tensor_load(tmp_path / "r.ouro", packed=True), packed.ravel())


def test_errors(tmp_path):
    with pytest.raises(ob.IoError, match="cannot open"):
        ob.tensor_load(tmp_path / "missing.ouro")
    (tmp_path / "bad.ouro").write_bytes(b"NOPE" + bytes(20))
    with pytest.raises(ob.IoError, match="bad magic"):
        ob.tensor_load(tmp_path / "bad.ouro")
    ob.tensor_save(tmp_path / "t.ouro", np.ones((4, 4)), ob.DTYPE_F64)
    raw = (tmp_path / "t.ouro").read_bytes()
    (tmp_path / "trunc.ouro").write_bytes(raw[:-8])
    with pytest.raises(ob.IoError, match="truncated"):
        ob.tensor_load(tmp_path / "trunc.ouro")
    import ctypes as C
    lib = ob.load()
    out = np.zeros(16, np.int8)
    st = lib.ouro_b200_tensor_load(str(tmp_path / "t.ouro").encode(), ob.DTYPE_I8, out.ctypes.data_as(C.c_void_p),
                                   out.nbytes, 0)
    assert st == 4 and b"dtype mismatch" in lib.ouro_b200_last_error()
    with pytest.raises(ob.ValidationError, match="outside"):
        ob.tensor_save(tmp_path / "x.ouro", np.array([8], np.int8), ob.DTYPE_U4)
    assert not os.path.exists(tmp_path / "x.ouro")
