"""Tiny workload for compute-sanitizer (racecheck / synccheck / memcheck, one
tool per gpurun call): the TMA codec kernels (step_tma_kernel), the generic
step kernel (unaligned pointers), the lossless codec, and the NVLink
engine's fused ring and one-shot kernels as virtual ranks on one GPU, each
checked against the CPU oracle so a run that passes is also correct.

  compute-sanitizer --tool racecheck python tools/sanitize_case.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import hccx_util as U  # noqa: E402
import oracle_lib as O  # noqa: E402

ok = True
n = 1 << 16
x = O.fill(3, "normal", n, 1e-3)
for kind, rate in (("fixed-rate", 8), ("fixed-rate", 5), ("zfp-rate", 8), ("identity", 0)):
    for off in (0, 1):  # aligned (TMA kernel) and unaligned (generic kernel)
        pay, st = U.compress(kind, rate, x, in_off=off, out_off=off)
        want = O.fr_compress(rate, x) if kind == "fixed-rate" else (
            O.zfp_compress(rate, x) if kind == "zfp-rate" else x.view(np.uint8))
        ok &= st == 0 and pay.tobytes() == want.tobytes()
        dec = U.decompress(kind, rate, pay, n, in_off=off, out_off=off)
        ok &= dec.tobytes() == (O.fr_decompress(rate, want, n) if kind == "fixed-rate" else (
            O.zfp_decompress(rate, want, n) if kind == "zfp-rate" else x)).tobytes()
print("codec ok" if ok else "codec FAIL", flush=True)

os.environ["HCCX_ONESHOT_BYTES"] = "0"
m = U.MComm(2, 1 << 15)
xs = np.stack([O.fill(10 + j, "uniform", 2 * 6144 + 512) for j in range(2)])
got, st = m.allreduce(xs, "fixed-rate", 8, True)
want, _ = O.allreduce(xs, "fixed-rate", 8, True)
ok &= st == 0 and got.tobytes() == want.tobytes()
os.environ["HCCX_ONESHOT_BYTES"] = str(1 << 40)
got, st = m.allreduce(xs, "fixed-rate", 8, False)
want, _ = O.allreduce(xs, "fixed-rate", 8, False)
ok &= st == 0 and got.tobytes() == want.tobytes()
got, st = m.allreduce(xs, "lossless", 0, False)
want, _ = O.allreduce(xs, "lossless", 0, False)
ok &= st == 0 and got.tobytes() == want.tobytes()
print("SANITIZE CASE OK" if ok else "SANITIZE CASE FAIL", flush=True)
sys.exit(0 if ok else 1)
