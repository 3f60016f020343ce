"""The plane-at-a-time zfp coder (csrc/zfp_planes.cuh, shared by the device
codec) against the published per-bit loops, exhaustively (CPU, g++)."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_plane_coder_matches_per_bit_loops(tmp_path):
    exe = tmp_path / "test_zfp_planes"
    subprocess.run(["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "paper_2409_02423_b200", "csrc"),
                    os.path.join(ROOT, "tests", "cpp", "test_zfp_planes.cpp"), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "0 failures" in out.stdout
