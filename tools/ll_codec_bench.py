"""Framed LosslessPredictor message codec on one GPU (the per-hop work of
the lossless collectives): hccx_lossless_frame_encode / _decode (fold) of
smooth and random fp32, CUDA-event time per call.

  python tools/ll_codec_bench.py [n ...]
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_02423_b200 import _lib  # noqa: E402

sizes = [int(a) for a in sys.argv[1:]] or [1 << 20, 1 << 22, 1 << 24]
K = int(os.environ.get("LL_K", "10"))
torch.cuda.set_device(0)
s = torch.cuda.current_stream()


def timed(fn):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(K):
        fn()
    b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / K * 1e3


for n in sizes:
    for kind in ("smooth", "random"):
        if kind == "smooth":
            t = torch.arange(n, device="cuda", dtype=torch.float32)
            x = ((torch.sin(t * 1e-4) * 1e-2) * 4096).round() / 4096
        else:
            x = torch.randn(n, device="cuda")
        cap = int(_lib.hccx_lossless_frame_max_bytes(n))
        msg = torch.zeros(cap, dtype=torch.uint8, device="cuda")
        out = torch.zeros(n, device="cuda")
        sp = s.cuda_stream
        enc = timed(lambda: _lib.hccx_lossless_frame_encode(x.data_ptr(), n, msg.data_ptr(), cap, sp))
        dec = timed(lambda: _lib.hccx_lossless_frame_decode(msg.data_ptr(), cap, n, out.data_ptr(), 1, sp))
        assert _lib.hccx_frame_status(sp) == 0
        container = int(msg[:8].cpu().numpy().view("u8")[0])
        print(json.dumps({"values": n, "data": kind, "payload": container - 18, "ratio": round(4 * n / (container - 18), 3),
                          "encode_us": round(enc, 1), "decode_fold_us": round(dec, 1),
                          "encode_GBps": round(4 * n / enc / 1e3, 1), "decode_GBps": round(4 * n / dec / 1e3, 1)}),
              flush=True)
