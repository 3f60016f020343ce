#!/usr/bin/env python
"""Benchmark of the compressed-collective hot path on B200.

Metric (BASELINE.json): "compressed allreduce effective GB/s (uncompressed
bytes/s) at 8xB200; codec GB/s vs HBM".

  N = 1  -> workload "codec-roundtrip": BASELINE config 1, the largest
            single-GPU configuration: fixed-rate compress + decompress of 2^24
            synthetic fp32 gradient values at rate 8.  value = 4n / step time.
  N > 1  -> workload "allreduce": BASELINE config 2, a 256 MiB fp32 gradient
            bucket per rank, compressed ring allreduce at rate 8 through the
            NVLink engine (one process per GPU, launched by torchrun).  value
            = 4n / step time (algbw convention, the same for the uncompressed
            NCCL allreduce reported beside it).

`--impl reference` times the reference's own CPU implementation of the same
workload (oracle/_ref = /root/reference/proj compiled unmodified; the C
restatement oracle/ when _ref is absent) on the host cores.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "compressed allreduce effective GB/s (uncompressed bytes/s) at 8xB200; codec GB/s vs HBM"
L2_BYTES = 126 * 1024 * 1024


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


# --------------------------------------------------------------- clocks ----

class ClockSampler:
    """SM clock and throttle reasons sampled (NVML, every ~2 ms) while the
    timed region runs; the summary goes into the JSON line's "clocks"."""

    REASONS = {  # nvmlClocksEventReason* bits
        0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap",
    }

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.stop = threading.Event()
        self.t = None

    def __enter__(self):
        try:
            import pynvml as N

            N.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[self.device]) if vis else self.device
            self.h = N.nvmlDeviceGetHandleByIndex(idx)
            self.N = N
            self.max_sm = N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM)
            self._sample()
            self.t = threading.Thread(target=self._loop, daemon=True)
            self.t.start()
        except Exception:
            self.t = None
        return self

    def _sample(self):
        N = self.N
        sm = N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM)
        try:
            r = N.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        except Exception:
            r = N.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
        self.rows.append((sm, r))

    def _loop(self):
        while not self.stop.is_set():
            try:
                self._sample()
            except Exception:
                return
            time.sleep(0.002)

    def __exit__(self, *exc):
        if self.t:
            self.stop.set()
            self.t.join(timeout=2)
            try:
                self._sample()
            except Exception:
                pass

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm = sorted(r[0] for r in self.rows)
        reasons = sorted({name for _, bits in self.rows for b, name in self.REASONS.items() if bits & b})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": self.max_sm, "reasons": reasons,
                "samples": len(self.rows)}


def traffic_for(kernel_tag: str):
    """dram read+write bytes per launch from the committed ncu --set full
    summary (profiles/traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f).get(kernel_tag)
    except Exception:
        return None


# ---------------------------------------------------------- CPU baselines --

def _cpu_lib():
    """(ctypes lib, kind): the reference compiled from its own sources, else the
    C restatement.  Only the CPU-baseline legs touch oracle/."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_lib as O  # noqa: E402

    return O, ("reference" if O.ref is not None else "port")


def cpu_codec_roundtrip(n: int, rate: int, reps: int):
    """Seconds per compress+decompress round trip of n values on the host."""
    import numpy as np

    O, kind = _cpu_lib()
    x = O.fill(1234, "normal", n, 1e-3)
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        if kind == "reference":
            payload, cc = O.ref_compress("fixed-rate", rate, x)
            O.ref_decompress("fixed-rate", rate, payload, n, cc)
        else:
            p = O.fr_compress(rate, x)
            O.fr_decompress(rate, p, n)
        times.append(time.perf_counter() - t0)
    del np
    return sorted(times)[len(times) // 2], kind


def cpu_allreduce(p: int, n: int, rate: int, reps: int):
    import numpy as np

    O, kind = _cpu_lib()
    x = np.stack([O.fill(1234 + j, "normal", n, 1e-3) for j in range(p)])
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        if kind == "reference":
            O.ref_allreduce(x, "fixed-rate", rate, False)
        else:
            O.allreduce(x, "fixed-rate", rate, False)
        times.append(time.perf_counter() - t0)
    return sorted(times)[len(times) // 2], kind


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# --------------------------------------------------------- N = 1: codec ----

def bench_codec(args):
    import numpy as np
    import torch

    from paper_2409_02423_b200 import _lib

    torch.cuda.set_device(0)
    n, rate = args.n or (1 << 24), args.rate
    codec = _lib.Codec(2, rate)
    wire = C.c_uint64()
    assert _lib.hccx_wire_size_bytes(codec, n, C.byref(wire)) == 0
    W = wire.value
    per_set = 4 * n + W + 4 * n
    nsets = max(2, -(-3 * L2_BYTES // per_set))  # rotate so every step touches cold data
    g = torch.Generator(device="cuda").manual_seed(1234)
    xs = [(torch.randn(n, device="cuda", generator=g) * 1e-3) for _ in range(nsets)]
    ps = [torch.empty(W, dtype=torch.uint8, device="cuda") for _ in range(nsets)]
    ys = [torch.empty(n, device="cuda") for _ in range(nsets)]
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream()
    sp = s.cuda_stream

    def step(i, stream, which=3):
        k = i % nsets
        st = 0
        if which & 1:
            st |= _lib.hccx_compress(codec, xs[k].data_ptr(), n, ps[k].data_ptr(), err.data_ptr(), stream)
        if which & 2:
            st |= _lib.hccx_decompress(codec, ps[k].data_ptr(), W, n, ys[k].data_ptr(), stream)
        assert st == 0

    for i in range(args.warmup):
        step(i, sp)
    assert _lib.hccx_flag_status(err.data_ptr(), sp) == 0
    torch.cuda.synchronize()

    # The K timed steps are captured once into a CUDA graph (launch-bound
    # inner loop -> graph, no host issue gaps or per-kernel events between
    # the kernels) and replayed inside the timed region.
    def capture(which, count):
        g = torch.cuda.CUDAGraph()
        cs = torch.cuda.Stream()
        cs.wait_stream(s)
        with torch.cuda.stream(cs):
            g.capture_begin()
            for i in range(count):
                step(i, cs.cuda_stream, which)
            g.capture_end()
        torch.cuda.synchronize()
        return g

    launches0 = _lib.hccx_launch_count()
    g_steps = capture(3, args.steps)
    launches = _lib.hccx_launch_count() - launches0
    g_steps.replay()  # upload + one untimed pass
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(0) as clk:
        torch.cuda.synchronize()
        t0.record(s)
        g_steps.replay()
        t1.record(s)
        torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / args.steps

    # Per-kernel average launch duration (roofline): K back-to-back launches
    # of one kernel over the same rotated buffers, one event pair around the
    # replay, on the stream the kernels run on.
    def kernel_ms(which):
        g = capture(which, args.steps)
        g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        g.replay()
        b.record(s)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / args.steps

    tc, td = kernel_ms(1), kernel_ms(2)
    # correctness of the timed output: decompress(compress(x)) within the block bound
    k = (args.steps - 1) % nsets
    assert torch.isfinite(ys[k]).all()

    hbm, peak_src = peaks()
    alg = 4 * n + W  # per launch, both kernels
    dom = ("compress", tc) if tc >= td else ("decompress", td)
    achieved = alg / (dom[1] * 1e-3) / 1e9

    # e2e: the reference-facing host-buffer API (hccx_compress_host /
    # hccx_decompress_host), pinned host buffers, copies inside the region.
    hx = torch.empty(n, dtype=torch.float32, pin_memory=True)
    hx.copy_(xs[0].cpu())
    hp = torch.empty(W, dtype=torch.uint8, pin_memory=True)
    hy = torch.empty(n, dtype=torch.float32, pin_memory=True)
    for _ in range(2):
        assert _lib.hccx_compress_host(codec, hx.data_ptr(), n, hp.data_ptr(), 0) == 0
        assert _lib.hccx_decompress_host(codec, hp.data_ptr(), W, n, hy.data_ptr(), 0) == 0
    e2e_steps = max(3, min(args.steps, 20))
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    for _ in range(e2e_steps):
        assert _lib.hccx_compress_host(codec, hx.data_ptr(), n, hp.data_ptr(), 0) == 0
        assert _lib.hccx_decompress_host(codec, hp.data_ptr(), W, n, hy.data_ptr(), 0) == 0
    torch.cuda.synchronize()
    e2e_s = (time.perf_counter() - w0) / e2e_steps

    # CPU baseline: the reference's own codec on this host, bounded sample.
    cpu_s, cpu_kind = cpu_codec_roundtrip(n, rate, reps=3)
    del np

    line = {
        "metric": METRIC,
        "value": round(4 * n / (ms * 1e-3) / 1e9, 2),
        "unit": "GB/s",
        "n_gpus": 1,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms, 5),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic (torch.randn * 1e-3 fp32 gradient-like values, seed 1234)",
        "config": {
            "workload": "codec-roundtrip: fixed-rate compress + decompress (BASELINE config 1)",
            "n_values": n, "rate_bits": rate, "payload_bytes": W,
            "l2": f"inputs rotated over {nsets} buffer sets ({nsets * per_set >> 20} MiB > 126 MiB L2)",
            "compress_ms": round(tc, 5), "decompress_ms": round(td, 5),
            "timing": "K steps captured in one CUDA graph, events around the replay; per-kernel ms from K "
                      "back-to-back launches of that kernel alone",
            "compress_GBps_uncompressed": round(4 * n / (tc * 1e-3) / 1e9, 1),
            "decompress_GBps_uncompressed": round(4 * n / (td * 1e-3) / 1e9, 1),
        },
        "roofline": {
            "bound": "hbm", "kernel": dom[0], "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
            "frac": round(achieved / hbm, 4), "peak_source": peak_src,
            "algorithmic_bytes_per_launch": alg, "traffic": traffic_for(dom[0]),
        },
        "cpu_baseline": {
            "value": round(4 * n / cpu_s / 1e9, 4), "unit": "GB/s", "cores": host_threads() if cpu_kind ==
            "reference" else 1, "kind": cpu_kind,
            "sample": f"full workload: {n} values, fixed-rate:{rate} compress+decompress, median of 3",
        },
        "e2e": {
            "value": round(4 * n / e2e_s / 1e9, 3), "unit": "GB/s", "h2d_bytes_per_step": 4 * n + W,
            "d2h_bytes_per_step": W + 4 * n,
            "api": "hccx_compress_host + hccx_decompress_host (pinned host buffers)",
            "timer": "host wall clock around the synchronous host-buffer API, device synced both sides",
        },
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------- N > 1: allreduce ----

def bench_allreduce(args):
    from paper_2409_02423_b200 import dist

    dist.bench_allreduce_main(args, METRIC, ClockSampler, peaks, traffic_for, cpu_allreduce, host_threads)


# ------------------------------------------------------- reference arm ----

def bench_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    n_gpus = args.gpus
    rate = args.rate
    threads = host_threads()
    if n_gpus <= 1:
        n = args.n or (1 << 24)
        sample = f"full workload: {n} values, fixed-rate:{rate} compress+decompress (OpenMP, {threads} threads)"
        run = lambda: cpu_codec_roundtrip(n, rate, reps=1)  # noqa: E731
        units = 4 * n
        workload = "codec-roundtrip: fixed-rate compress + decompress (BASELINE config 1)"
    else:
        p = n_gpus
        n = args.ref_n or (1 << 22)
        sample = (f"bounded sample: hcc::allreduce of {n} values per rank (of 2^26), p={p}, all ranks "
                  f"simulated in one process (reference design), fixed-rate:{rate}")
        run = lambda: cpu_allreduce(p, n, rate, reps=1)  # noqa: E731
        units = 4 * n
        workload = "allreduce (BASELINE config 2), bounded sample"
    for _ in range(args.warmup):
        run()
    ts = []
    kind = "port"
    for _ in range(args.steps):
        t, kind = run()
        ts.append(t)
    sec = sum(ts) / len(ts)
    value = round(units / sec / 1e9, 5)
    line = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": n_gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(sec * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic (hcc::Rng normal * 1e-3)",
        "config": {"workload": workload, "rate_bits": rate, "world_size": world},
        "impl": "reference",
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": threads if kind == "reference" else 1,
                         "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="hccx", choices=["hccx", "reference"])
    ap.add_argument("--rate", type=int, default=8)
    ap.add_argument("--n", type=int, default=0, help="values per rank (default: the BASELINE config size)")
    ap.add_argument("--ref-n", type=int, default=0, help="reference-arm sample size per rank (N>1)")
    ap.add_argument("--nccl", type=int, default=1, help="also time an uncompressed NCCL allreduce (N>1)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        bench_reference(args)
        return
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1 or args.gpus > 1:
        bench_allreduce(args)
    else:
        bench_codec(args)


if __name__ == "__main__":
    main()
