"""Reference-format LosslessPredictor decode (hccx_lossless_decompress: the
bare payload, no chunk offsets) on one GPU: smooth / sparse / random fp32,
CUDA-event time per call.  An ncu launch list of this script splits the
offset search (jump rounds, chunk walk) from the decode.

  python tools/ll_ref_decode.py [n]
"""
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_02423_b200 import _lib  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 24
K = int(os.environ.get("LL_K", "3"))
torch.cuda.set_device(0)
s = torch.cuda.current_stream()
for kind in ("smooth", "sparse", "random"):
    if kind == "smooth":
        t = torch.arange(n, device="cuda", dtype=torch.float32)
        x = ((torch.sin(t * 1e-4) * 1e-2) * 4096).round() / 4096
    elif kind == "sparse":
        x = torch.randn(n, device="cuda") * (torch.rand(n, device="cuda") < 0.1)
    else:
        x = torch.randn(n, device="cuda")
    cap = int(_lib.hccx_lossless_max_bytes(n))
    pay = torch.empty(cap, dtype=torch.uint8, device="cuda")
    nb = C.c_uint64()
    assert _lib.hccx_lossless_compress(x.data_ptr(), n, pay.data_ptr(), cap, C.byref(nb), s.cuda_stream) == 0
    y = torch.empty(n, device="cuda")
    assert _lib.hccx_lossless_decompress(pay.data_ptr(), nb.value, n, y.data_ptr(), s.cuda_stream) == 0
    torch.cuda.synchronize()
    assert torch.equal(y.view(torch.int32), x.view(torch.int32))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(K):
        _lib.hccx_lossless_decompress(pay.data_ptr(), nb.value, n, y.data_ptr(), s.cuda_stream)
    b.record(s)
    torch.cuda.synchronize()
    us = a.elapsed_time(b) / K * 1e3
    print(json.dumps({"data": kind, "values": n, "payload": nb.value, "ratio": round(4 * n / nb.value, 3),
                      "decompress_us": round(us, 1), "GBps": round(4 * n / us / 1e3, 2)}), flush=True)
