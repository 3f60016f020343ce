"""The C++ drop-in (namespace hcc, libhcc_b200.so) runs the reference's own
test cases (tests/cpp/test_hcc_shim.cpp) on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "test_hcc_shim")


def _build():
    subprocess.run(["make", "-C", os.path.join(ROOT, "paper_2409_02423_b200", "host")], check=True,
                   capture_output=True)


def test_shim_library_exports_reference_api():
    """CPU check: libhcc_b200.so exports the hcc:: entry points the reference
    header declares (mangled names), and links only libhccx for compute."""
    _build()
    so = os.path.join(ROOT, "paper_2409_02423_b200", "libhcc_b200.so")
    syms = subprocess.run(["nm", "-DC", so], capture_output=True, text=True, check=True).stdout
    for name in ("hcc::allreduce(", "hcc::ring_reduce_scatter(", "hcc::ring_allgather(", "hcc::p2p(",
                 "hcc::compress(", "hcc::decompress(", "hcc::wire_size_bytes(", "hcc::scheme_from_name(",
                 "hcc::to_bytes(", "hcc::from_bytes(", "hcc::build_layout(", "hcc::broadcast("):
        assert name in syms, name
    deps = subprocess.run(["ldd", so], capture_output=True, text=True).stdout
    assert "libhccx.so" in deps


@pytest.mark.gpu
def test_cpp_shim_reference_cases(cuda):
    _build()
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr[-3000:])
    assert r.returncode == 0 and " 0 failed" in r.stdout
