"""Codec kernel sweep on one GPU: per-kernel device time (CUDA events,
rotated buffers > L2) for rates x sizes.  Development tool; bench.py is the
contract."""
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_02423_b200 import _lib  # noqa: E402


def run(kind, rate, n, reps=50):
    codec = _lib.Codec(kind, rate)
    w = C.c_uint64()
    _lib.hccx_wire_size_bytes(codec, n, C.byref(w))
    W = w.value
    sets = max(2, -(-400 * 2 ** 20 // (8 * n + W)))
    xs = [torch.randn(n, device="cuda") * 1e-3 for _ in range(sets)]
    ps = [torch.empty(W, dtype=torch.uint8, device="cuda") for _ in range(sets)]
    ys = [torch.empty(n, device="cuda") for _ in range(sets)]
    s = torch.cuda.current_stream().cuda_stream
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3 * reps)]
    for i in range(5):
        _lib.hccx_compress(codec, xs[i % sets].data_ptr(), n, ps[i % sets].data_ptr(), None, s)
        _lib.hccx_decompress(codec, ps[i % sets].data_ptr(), W, n, ys[i % sets].data_ptr(), s)
    torch.cuda.synchronize()
    torch.cuda._sleep(int(4e6))  # let the host queue ahead of the GPU
    for i in range(reps):
        k = i % sets
        ev[3 * i].record()
        _lib.hccx_compress(codec, xs[k].data_ptr(), n, ps[k].data_ptr(), None, s)
        ev[3 * i + 1].record()
        _lib.hccx_decompress(codec, ps[k].data_ptr(), W, n, ys[k].data_ptr(), s)
        ev[3 * i + 2].record()
    torch.cuda.synchronize()
    tc = sorted(ev[3 * i].elapsed_time(ev[3 * i + 1]) for i in range(reps))[reps // 2]
    td = sorted(ev[3 * i + 1].elapsed_time(ev[3 * i + 2]) for i in range(reps))[reps // 2]
    alg = (4 * n + W) / 1e9
    return {"kind": kind, "rate": rate, "n": n, "compress_us": round(tc * 1e3, 2), "decompress_us": round(td * 1e3, 2),
            "compress_hbm_GBps": round(alg / (tc * 1e-3), 1), "decompress_hbm_GBps": round(alg / (td * 1e-3), 1)}


if __name__ == "__main__":
    torch.cuda.set_device(0)
    for kind, rates in ((2, [4, 8, 12, 16, 24, 32, 3, 7]), (0, [0]), (3, [8, 16])):
        for r in rates:
            for n in ([1 << 24, 1 << 26] if kind != 3 else [1 << 24]):
                print(json.dumps(run(kind, r, n)), flush=True)
