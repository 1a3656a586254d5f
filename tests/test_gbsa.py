"""CPU: GBSA instance files at the C ABI (tor_load_matrix / tor_save_matrix) against the
REFERENCE's own save_matrix / load_matrix_file (matrix_io.cpp:92-263), called through
oracle/_ref (the unmodified torfp sources).

- files the reference writes (text; binary 16 and 32 bit) load to the same doubles;
- files this library writes are byte-identical to the reference's;
- malformed files raise the same ParseError codes at the same positions.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

import paper_2009_01177_b200 as T
from paper_2009_01177_b200 import api
from paper_2009_01177_b200 import workloads as W
from paper_2009_01177_b200.matrix import load_matrix_bytes, save_matrix

ref = pytest.importorskip("oracle.ref")
if not ref.available():
    pytest.skip("oracle/_ref not built", allow_module_level=True)


def ref_save(m, fmt, bits=16):
    a00, a01 = m.interleaved()
    P = C.POINTER(C.c_double)
    size = C.c_size_t()
    code, msg, mask, row = ref._err()
    L = ref.lib()
    st = L.ref_save_matrix(C.c_int(m.n_modes), a00.ctypes.data_as(P), a01.ctypes.data_as(P),
                           C.c_int(fmt == "binary"), C.c_int(bits), None, C.c_size_t(0), C.byref(size), code, 64,
                           msg, 256, C.byref(mask), C.byref(row))
    if st:
        raise ref.RefError(st, code.value.decode(), msg.value.decode())
    buf = C.create_string_buffer(size.value)
    L.ref_save_matrix(C.c_int(m.n_modes), a00.ctypes.data_as(P), a01.ctypes.data_as(P), C.c_int(fmt == "binary"),
                      C.c_int(bits), buf, C.c_size_t(size.value), C.byref(size), code, 64, msg, 256, C.byref(mask),
                      C.byref(row))
    return buf.raw[: size.value]


def ref_load(b: bytes):
    n, bits = C.c_int(), C.c_int()
    code, msg, mask, row = ref._err()
    L = ref.lib()
    cap = 4096 * 4097 // 2
    st = L.ref_load_matrix(b, C.c_size_t(len(b)), C.byref(n), C.byref(bits), None, None, C.c_size_t(0), code, 64,
                           msg, 256, C.byref(mask), C.byref(row))
    if st:
        return dict(status=st, code=code.value.decode(), position=row.value)
    t = n.value * (n.value + 1) // 2
    a00, a01 = np.zeros(2 * t), np.zeros(2 * t)
    P = C.POINTER(C.c_double)
    L.ref_load_matrix(b, C.c_size_t(len(b)), C.byref(n), C.byref(bits), a00.ctypes.data_as(P),
                      a01.ctypes.data_as(P), C.c_size_t(t), code, 64, msg, 256, C.byref(mask), C.byref(row))
    del cap
    return dict(status=0, n=n.value, bits=bits.value, a00=a00.view(np.complex128), a01=a01.view(np.complex128))


INSTANCES = [("gen5", lambda: T.generate_instance(5, 0.2, 0.05, 11)),
             ("gen12", lambda: T.generate_instance(12, 0.16, 0.06, 7)),
             ("cfg1", lambda: W.load_config_instance(1)),
             ("cfg4", lambda: W.load_config_instance(4))]


@pytest.mark.parametrize("name,make", INSTANCES)
@pytest.mark.parametrize("fmt,bits", [("text", 16), ("binary", 16), ("binary", 32)])
def test_reference_files_load_identically(name, make, fmt, bits):
    m = make()
    b = ref_save(m, fmt, bits)
    got = load_matrix_bytes(b)
    want = ref_load(b)
    assert want["status"] == 0
    assert got.n_modes == want["n"] and got.quant_bits == want["bits"]
    assert np.array_equal(got.a00, want["a00"]) and np.array_equal(got.a01, want["a01"])
    if fmt == "text":  # %.17g text is lossless
        assert np.array_equal(got.a00, m.a00) and np.array_equal(got.a01, m.a01)


@pytest.mark.parametrize("name,make", INSTANCES)
@pytest.mark.parametrize("fmt,bits", [("text", 16), ("binary", 16), ("binary", 32)])
def test_written_files_byte_identical(name, make, fmt, bits):
    m = make()
    assert save_matrix(m, fmt, bits) == ref_save(m, fmt, bits)


def _mutations():
    m = T.generate_instance(3, 0.2, 0.05, 3)
    txt = ref_save(m, "text")
    b16 = ref_save(m, "binary", 16)
    lines = txt.split(b"\n")
    yield "empty", b""
    yield "text magic", b"GBSA text 2\nmodes 3\n"
    yield "crlf ok", txt.replace(b"\n", b"\r\n")
    yield "blank lines ok", txt.replace(b"\n", b"\n\n")
    yield "no modes", lines[0] + b"\n"
    yield "bad modes", b"\n".join([lines[0], b"modes 0"] + lines[2:])
    yield "modes word", b"\n".join([lines[0], b"mode 3"] + lines[2:])
    yield "truncated entries", b"\n".join(lines[:7])
    yield "bad entry", b"\n".join(lines[:4] + [b"0.1 x"] + lines[5:])
    yield "range", b"\n".join(lines[:4] + [b"1.0 0.0"] + lines[5:])
    yield "nan", b"\n".join(lines[:4] + [b"nan 0.0"] + lines[5:])
    yield "bin short", b16[:5]
    yield "bin version", b16[:4] + b"\x02\x00" + b16[6:]
    yield "bin header", b16[:9]
    yield "bin bits", b16[:10] + b"\x08" + b16[11:]
    yield "bin dim", b16[:6] + b"\x00\x00\x00\x00" + b16[10:]
    yield "bin huge dim", b16[:6] + b"\x01\x10\x00\x00" + b16[10:]
    yield "bin truncated data", b16[:-1]
    yield "bin trailing ok", b16 + b"\x00\x01"
    yield "GBSA space -> text", b"GBSA text 1\nmodes 1\n0 0\n0 0\n"


@pytest.mark.parametrize("why,b", list(_mutations()), ids=[w for w, _ in _mutations()])
def test_malformed_files_same_errors(why, b):
    want = ref_load(b)
    if want["status"] == 0:
        got = load_matrix_bytes(b)
        assert np.array_equal(got.a00, want["a00"]) and np.array_equal(got.a01, want["a01"])
        return
    with pytest.raises(T.TorfpError) as e:
        load_matrix_bytes(b)
    assert e.value.code == want["code"], why
    assert isinstance(e.value, T.ParseError) == (want["status"] == 4)
    if want["status"] == 4:
        assert e.value.position == want["position"], why


def test_save_errors():
    m = T.generate_instance(3, 0.2, 0.05, 3)
    with pytest.raises(T.InvalidArgument) as e:
        save_matrix(m, "binary", 8)
    assert e.value.code == "matrixio/bits"
    big = T.InputMatrix(1, np.array([1.5 + 0j]), np.array([0j]))
    with pytest.raises(T.InvalidArgument) as e:
        save_matrix(big, "binary", 16)
    assert e.value.code == "matrixio/range"
    assert "tor_load_matrix" in api.EXPORTS and "tor_save_matrix" in api.EXPORTS
