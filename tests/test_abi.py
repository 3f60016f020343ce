"""The C ABI library loads and exports every symbol include/hccx.h declares;
pure host-side entry points (size laws, validation) answer without a GPU."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    src = open(os.path.join(ROOT, "include", "hccx.h")).read()
    return sorted(set(re.findall(r"^HCCX_API [^(]*?\b(hccx_\w+)\(", src, re.M)))


def test_header_declares_entry_points():
    names = declared()
    assert len(names) >= 25
    for must in ("hccx_compress", "hccx_decompress", "hccx_group_allreduce", "hccx_allreduce",
                 "hccx_reduce_scatter", "hccx_allgather", "hccx_broadcast", "hccx_p2p", "hccx_wire_size_bytes"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2409_02423_b200 import _lib

    for name in declared():
        assert hasattr(_lib.lib, name), name
    assert set(declared()) == set(_lib.EXPORTED)


def test_abi_version_and_strings():
    from paper_2409_02423_b200 import _lib

    assert _lib.hccx_abi_version() == 1
    assert _lib.hccx_status_string(1) == b"non-finite input value on a lossy path"


def _wire(kind, rate, n):
    from paper_2409_02423_b200 import _lib

    out = C.c_uint64()
    st = _lib.hccx_wire_size_bytes(_lib.Codec(kind, rate), n, C.byref(out))
    return st, out.value


def test_wire_size_law_kats():  # proj/tests/test_codec.cpp:110-116
    assert _wire(0, 0, 100) == (0, 400)
    assert _wire(2, 16, 64) == (0, 129)
    assert _wire(2, 8, 65) == (0, 130)
    assert _wire(2, 8, 0) == (0, 0)
    assert _wire(1, 0, 10)[0] == 3  # DataDependentSizeError
    assert _wire(2, 1, 10)[0] == 6  # InvalidSchemeError
    assert _wire(2, 33, 10)[0] == 6


@pytest.mark.parametrize("rate", range(2, 33))
def test_wire_size_matches_oracle(rate):
    import oracle_lib as O

    for n in (0, 1, 63, 64, 65, 10 ** 6, 2 ** 24, 2 ** 28 + 5):
        assert _wire(2, rate, n) == (0, O.wire_size("fixed-rate", rate, n))
        if rate >= 3:
            assert _wire(3, rate, n) == (0, O.wire_size("zfp-rate", rate, n))


def test_python_wire_size_errors():
    import paper_2409_02423_b200 as H

    assert H.wire_size_bytes(H.CodecSpec.fixed_rate(8), 1024) == 1040
    with pytest.raises(H.DataDependentSizeError):
        H.wire_size_bytes(H.CodecSpec.lossless(), 10)
