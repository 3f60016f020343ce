"""Kernel-variant timing (dev tool): for each HCCX_LIB build given on the
command line, time fixed-rate compress/decompress at 2^24 and 2^26 values
(rate 8) in a subprocess, next to torch copy / sum of the same bytes as a
small-transfer HBM calibration."""
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))


def child():
    import torch

    sys.path.insert(0, HERE)
    from codec_sweep import run

    torch.cuda.set_device(0)
    out = {"lib": os.environ.get("HCCX_LIB", "default")}
    for n in (1 << 24, 1 << 26):
        r = run(2, int(os.environ.get("RATE", "8")), n)
        out[f"c{n.bit_length() - 1}"] = r["compress_us"]
        out[f"d{n.bit_length() - 1}"] = r["decompress_us"]
    if os.environ.get("CALIB"):
        for n in (1 << 24, 1 << 26):
            xs = [torch.randn(n, device="cuda") for _ in range(8)]
            ys = [torch.empty(n, device="cuda") for _ in range(8)]
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            for i in range(5):
                ys[i % 8].copy_(xs[i % 8])
            torch.cuda.synchronize()
            torch.cuda._sleep(int(2e6))
            a.record()
            for i in range(40):
                ys[i % 8].copy_(xs[i % 8])
            b.record()
            torch.cuda.synchronize()
            out[f"copy{n.bit_length() - 1}_us"] = round(a.elapsed_time(b) / 40 * 1e3, 2)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--child":
        child()
        sys.exit(0)
    libs = sys.argv[1:] or [""]
    for i, lib in enumerate(libs):
        env = dict(os.environ)
        if lib:
            env["HCCX_LIB"] = os.path.abspath(lib)
        if i == 0:
            env["CALIB"] = "1"
        subprocess.run([sys.executable, __file__, "--child"], env=env, check=False)
