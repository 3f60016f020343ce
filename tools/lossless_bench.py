"""LosslessPredictor device codec throughput (dev tool): 2^24 values, dense
(normal*1e-3: every chunk falls back to raw) and sparse (90% zeros: coded),
compress (size pass + scan + emit) and decompress (offset walk + decode),
wall time around the synchronising C calls, median of 10."""
import ctypes as C
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_02423_b200 import _lib  # noqa: E402

torch.cuda.set_device(0)
n = 1 << 24
for name in ("dense", "sparse", "smooth"):
    g = torch.Generator(device="cuda").manual_seed(5)
    if name == "dense":
        x = torch.randn(n, device="cuda", generator=g) * 1e-3
    elif name == "sparse":
        x = torch.randn(n, device="cuda", generator=g) * (torch.rand(n, device="cuda", generator=g) < 0.1)
    else:
        x = torch.arange(n, device="cuda", dtype=torch.float32).div_(1 << 12).floor_()
    cap = _lib.hccx_lossless_max_bytes(n)
    out = torch.empty(cap, dtype=torch.uint8, device="cuda")
    back = torch.empty_like(x)
    nb = C.c_uint64()
    s = torch.cuda.current_stream().cuda_stream
    tc, td = [], []
    for i in range(12):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        assert _lib.hccx_lossless_compress(x.data_ptr(), n, out.data_ptr(), cap, C.byref(nb), s) == 0
        t1 = time.perf_counter()
        assert _lib.hccx_lossless_decompress(out.data_ptr(), nb.value, n, back.data_ptr(), s) == 0
        t2 = time.perf_counter()
        if i >= 2:
            tc.append(t1 - t0)
            td.append(t2 - t1)
    assert torch.equal(back.view(torch.int32), x.view(torch.int32))
    tc.sort(), td.sort()
    print(json.dumps({"data": name, "n": n, "payload_bytes": nb.value, "ratio": round(4 * n / nb.value, 3),
                      "compress_us": round(tc[5] * 1e6, 1), "decompress_us": round(td[5] * 1e6, 1),
                      "compress_GBps": round(4 * n / tc[5] / 1e9, 1), "decompress_GBps": round(4 * n / td[5] / 1e9, 2)}),
          flush=True)
