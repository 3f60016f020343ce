#!/usr/bin/env python
"""Benchmark of the compressed-collective hot path on B200.

Metric (BASELINE.json): "compressed allreduce effective GB/s (uncompressed
bytes/s) at 8xB200; codec GB/s vs HBM".

  N = 1  -> workload "codec-roundtrip": BASELINE config 1, the largest
            single-GPU configuration: fixed-rate compress + decompress of 2^24
            synthetic fp32 gradient values at rate 8.  value = 4n / step time.
  N > 1  -> workload "allreduce": BASELINE config 2, a 256 MiB fp32 gradient
            bucket per rank, compressed ring allreduce at rate 8 through the
            NVLink engine (one process per GPU).  value = 4n / step time (algbw
            convention, the same for the uncompressed NCCL allreduce reported
            beside it).  `python bench.py --gpus N` without torchrun re-launches
            itself under torch.distributed.run with N local ranks.

Inputs are the reference's hcc::Rng streams (1e-3 * normal(), seed 1234 +
rank; include/hcc/rng.hpp), the same buffers the CPU reference sees.

`--impl reference` times the reference's own CPU implementation of the same
workload (oracle/_ref = /root/reference/proj compiled unmodified; the C
restatement oracle/ when _ref is absent) on the host cores, with the same
`config` dict as this arm.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import socket
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "compressed allreduce effective GB/s (uncompressed bytes/s) at 8xB200; codec GB/s vs HBM"
L2_BYTES = 126 * 1024 * 1024
NVLINK_PEAK = 770.0  # GB/s per direction per GPU: measured peer copy (B200_PROFILING.md; 900 nominal)
NVLINK_NOMINAL = 900.0
SOAK_S = 0.15        # clock-record region (seconds of back-to-back steps) before the timed K steps


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def workload_config(n_gpus: int, n: int, rate: int) -> dict:
    """The `config` dict: identical for this arm and --impl reference."""
    if n_gpus <= 1:
        return {"workload": "codec-roundtrip: fixed-rate compress + decompress (BASELINE config 1)",
                "n_values": n, "rate_bits": rate, "parallelism": "single-gpu"}
    return {"workload": "allreduce: compressed ring allreduce, Sum, of a 256 MiB fp32 bucket per rank "
                        "(BASELINE config 2)", "n_values_per_rank": n, "rate_bits": rate,
            "parallelism": f"dp{n_gpus}"}


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


# ------------------------------------------------------------ inputs -------

def synth(seed: int, n: int, scale: float = 1e-3):
    """hcc::Rng(seed) stream of scale * normal() (libhcc_b200.so, include/hcc/rng.hpp)."""
    import numpy as np

    lib = C.CDLL(os.path.join(ROOT, "paper_2409_02423_b200", "libhcc_b200.so"))
    lib.hcc_b200_fill.argtypes = [C.c_uint64, C.c_int, C.c_uint64, C.c_float, C.c_float, C.c_void_p]
    lib.hcc_b200_fill.restype = None
    x = np.empty(n, np.float32)
    lib.hcc_b200_fill(seed, 0, n, scale, 0.0, x.ctypes.data)
    return x


# ---------------------------------------------------------- CPU baselines --

def _cpu_lib():
    """(ctypes lib, kind): the reference compiled from its own sources, else the
    C restatement.  Only the CPU-baseline legs and the parity checker touch
    oracle/."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_lib as O  # noqa: E402

    # torchrun exports OMP_NUM_THREADS=1 to every rank; the reference's
    # OpenMP codec gets all host threads here (libgomp of oracle/_ref)
    try:
        C.CDLL("libgomp.so.1").omp_set_num_threads(host_threads())
    except OSError:
        pass
    return O, ("reference" if O.ref is not None else "port")


def cpu_codec_roundtrip(n: int, rate: int, reps: int, x=None):
    """Seconds per compress+decompress round trip of n values on the host."""
    O, kind = _cpu_lib()
    x = synth(1234, n) if x is None else x
    if kind == "reference":  # only the reference library's own calls are timed
        return O.ref_time_codec("fixed-rate", rate, x, reps), kind
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        p = O.fr_compress(rate, x)
        O.fr_decompress(rate, p, n)
        times.append(time.perf_counter() - t0)
    return sorted(times)[len(times) // 2], kind


def cpu_allreduce(x, rate: int, reps: int):
    """Seconds per hcc::allreduce of the [p, n] inputs x (all p ranks
    simulated in one process: the reference design)."""
    O, kind = _cpu_lib()
    if kind == "reference":  # only hcc::allreduce itself is timed
        return O.ref_time_allreduce(x, "fixed-rate", rate, reps), kind
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        O.allreduce(x, "fixed-rate", rate, False)
        times.append(time.perf_counter() - t0)
    return sorted(times)[len(times) // 2], kind


def pinned_local(device: int, shapes):
    """Pinned host buffers for the e2e copies, allocated while this process
    runs on the CPUs NVML reports as local to `device`, so their pages sit on
    the GPU's own NUMA node (first touch); the previous CPU affinity is
    restored afterwards (the CPU baseline keeps every host thread).
    shapes: [(numel, dtype)].  Returns (buffers, note)."""
    import torch

    before = os.sched_getaffinity(0)
    note = "pinned pages allocated on the launching CPUs"
    try:
        import pynvml

        pynvml.nvmlInit()
        pynvml.nvmlDeviceSetCpuAffinity(pynvml.nvmlDeviceGetHandleByIndex(device))
        note = f"pinned pages first-touched on gpu {device}'s NVML-local CPUs ({len(os.sched_getaffinity(0))})"
    except Exception:
        pass
    try:
        bufs = [torch.empty(k, dtype=dt, pin_memory=True) for k, dt in shapes]
    finally:
        os.sched_setaffinity(0, before)
    return bufs, note


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# --------------------------------------------------------- N = 1: codec ----

def bench_codec(args):
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
    x0 = synth(1234, n)
    base = torch.from_numpy(x0).cuda()
    # buffer set k holds the same stream rotated by k blocks-of-256 (distinct
    # addresses and contents, identical statistics)
    xs = [torch.roll(base, 256 * k) for k in range(nsets)]
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
        # clock record: >= SOAK_S of the same replays right before the timed
        # region (the K steps alone last well under a millisecond)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        g_steps.replay()
        b.record(s)
        torch.cuda.synchronize()
        reps = max(1, int(SOAK_S / max(a.elapsed_time(b) * 1e-3, 1e-6)))
        a.record(s)
        for _ in range(reps):
            g_steps.replay()
        b.record(s)
        torch.cuda.synchronize()
        soak_ms = a.elapsed_time(b) / (reps * args.steps)
        torch.cuda.nvtx.range_push("bench_timed")  # ncu --nvtx --nvtx-include bench_timed/ (launch list)
        t0.record(s)
        g_steps.replay()
        t1.record(s)
        torch.cuda.nvtx.range_pop()
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

    # Checker (outside the timed region): the timed step's payload and
    # decoded values vs the CPU oracle on the same input, bit for bit.
    O, _ = _cpu_lib()
    k = (args.steps - 1) % nsets
    xk = xs[k].cpu().numpy()
    pay_ok = ps[k].cpu().numpy().tobytes() == O.fr_compress(rate, xk).tobytes()
    dec_ok = ys[k].cpu().numpy().tobytes() == O.fr_decompress(rate, O.fr_compress(rate, xk), n).tobytes()
    parity = {"checked": "timed step's payload and decoded values vs the CPU oracle (same input)",
              "payload_bit_exact": bool(pay_ok), "decoded_bit_exact": bool(dec_ok)}

    hbm, peak_src = peaks()
    alg = 4 * n + W  # per launch, both kernels
    dom = ("compress", tc) if tc >= td else ("decompress", td)
    achieved = alg / (dom[1] * 1e-3) / 1e9

    # e2e: the reference-facing host-buffer API (hccx_compress_host /
    # hccx_decompress_host), pinned host buffers, copies inside the region.
    (hx, hp, hy), numa_note = pinned_local(0, [(n, torch.float32), (W, torch.uint8), (n, torch.float32)])
    hx.copy_(torch.from_numpy(x0))
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

    # CPU baseline: the reference's own codec on this host, same input.
    cpu_s, cpu_kind = cpu_codec_roundtrip(n, rate, reps=3, x=x0)

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
        "data": "synthetic (hcc::Rng(1234) 1e-3*normal() fp32 gradient-like values, the reference's stream)",
        "config": workload_config(1, n, rate),
        "detail": {
            "payload_bytes": W,
            "l2": f"inputs rotated over {nsets} buffer sets ({nsets * per_set >> 20} MiB > 126 MiB L2)",
            "compress_ms": round(tc, 5), "decompress_ms": round(td, 5),
            "timing": "K steps captured in one CUDA graph, events around the replay; per-kernel ms from K "
                      "back-to-back launches of that kernel alone",
            "clock_soak": f"{reps} replays of the K-step graph ({reps * args.steps * soak_ms:.0f} ms) right before "
                          f"the timed replay, sampled with the clocks",
            "soak_GBps": round(4 * n / (soak_ms * 1e-3) / 1e9, 2),
            "compress_GBps_uncompressed": round(4 * n / (tc * 1e-3) / 1e9, 1),
            "decompress_GBps_uncompressed": round(4 * n / (td * 1e-3) / 1e9, 1),
        },
        "parity": parity,
        "roofline": {
            "bound": "hbm", "kernel": dom[0], "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
            "frac": round(achieved / hbm, 4), "peak_source": peak_src,
            "algorithmic_bytes_per_launch": alg, "traffic": traffic_for(dom[0]),
        },
        "cpu_baseline": {
            "value": round(4 * n / cpu_s / 1e9, 4), "unit": "GB/s", "cores": host_threads() if cpu_kind ==
            "reference" else 1, "kind": cpu_kind,
            "sample": f"full workload: {n} values, fixed-rate:{rate} compress+decompress of the same input, "
                      f"median of 3",
        },
        "e2e": {
            "value": round(4 * n / e2e_s / 1e9, 3), "unit": "GB/s", "h2d_bytes_per_step": 4 * n + W,
            "d2h_bytes_per_step": W + 4 * n,
            "api": "hccx_compress_host + hccx_decompress_host (pinned host buffers)",
            "host_buffers": numa_note,
            "timer": "host wall clock around the synchronous host-buffer API, device synced both sides",
        },
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)
    if not (pay_ok and dec_ok):
        sys.exit("bench: timed output differs from the CPU oracle")


# ----------------------------------------------------- N > 1: allreduce ----

def bench_allreduce(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2409_02423_b200 import _lib
    from paper_2409_02423_b200.codec import CodecSpec, wire_size_bytes
    from paper_2409_02423_b200.dist import NvlinkComm

    # the image exports NCCL_DEBUG=VERSION, and NCCL prints its version line
    # on stdout at VERSION and WARN levels: keep stdout to the one JSON line
    # (NCCL's own log of the baseline is tools/nccl_info.py)
    if os.environ.get("NCCL_DEBUG", "").upper() in ("VERSION", "WARN"):
        os.environ.pop("NCCL_DEBUG")
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    rank, world = dist.get_rank(), dist.get_world_size()
    n = args.n or (1 << 26)  # 256 MiB fp32 per rank
    n -= n % (64 * world)    # whole 64-value blocks per chunk (sampled parity below)
    rate = args.rate
    spec = CodecSpec.fixed_rate(rate)
    comm = NvlinkComm(n)
    x_host = synth(1234 + rank, n)
    x = torch.from_numpy(x_host).cuda()
    out = torch.empty_like(x)
    s = torch.cuda.current_stream()

    def timed(fn, steps):
        import gc

        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()  # no fused kernel may be in flight across an NCCL call
        dist.barrier()
        torch.cuda.synchronize()
        gc.disable()  # a collection pause on one rank's host would stall every peer
        try:
            torch.cuda._sleep(int(1e6))
            t0.record(s)
            for _ in range(steps):
                fn()
            t1.record(s)
            torch.cuda.synchronize()
        finally:
            gc.enable()
        ms = torch.tensor([t0.elapsed_time(t1) / steps], device="cuda")
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        return float(ms.item())

    step = lambda: comm.allreduce(x, spec, 0, out)  # noqa: E731
    for _ in range(args.warmup):
        step()
    comm.status()
    with ClockSampler(local) as clk:
        per = timed(step, 3)
        soak = max(3, int(SOAK_S / max(per * 1e-3, 1e-6)))
        soak_ms = timed(step, soak)
        launches0 = _lib.hccx_launch_count()
        ms = timed(step, args.steps)
        launches = _lib.hccx_launch_count() - launches0
    comm.status()

    # Checker (outside the timed region): the 256 MiB output vs the CPU
    # oracle on sampled blocks: blocks are independent and
    # every chunk is whole blocks, so block b of every chunk of every rank is
    # itself an allreduce of n' = 64p values per rank with the same bits.
    c = n // world
    nb = c // 64
    rs = np.random.default_rng(7)
    blocks = sorted({0, nb - 1, nb // 2, *rs.choice(nb, size=min(nb, 61), replace=False).tolist()})
    idx = torch.tensor([i * c + 64 * b + k for b in blocks for i in range(world) for k in range(64)],
                       device="cuda", dtype=torch.int64)
    sample = torch.stack([x[idx], out[idx]])  # [2, S * p * 64]
    gathered = [torch.empty_like(sample) for _ in range(world)]
    dist.all_gather(gathered, sample)
    parity = None
    if rank == 0:
        O, _ = _cpu_lib()
        S = len(blocks)
        g = torch.stack(gathered).cpu().numpy().reshape(world, 2, S, world * 64)
        bad = 0
        for si in range(S):
            xin = np.ascontiguousarray(g[:, 0, si, :])
            want, _ = O.allreduce(xin, "fixed-rate", rate, False)
            if want.tobytes() != np.ascontiguousarray(g[:, 1, si, :]).tobytes():
                bad += 1
        parity = {"checked": f"{S} sampled 64-value blocks of every chunk on every rank of the timed output vs "
                             f"the CPU oracle allreduce of those blocks (n'=64p per rank)",
                  "blocks_bit_exact": S - bad, "blocks_checked": S, "bit_exact": bad == 0}
    # agreement: every rank holds bit-identical results
    h = torch.tensor([int(out.view(torch.int32).to(torch.int64).sum().item())], device="cuda")
    hs = [torch.zeros_like(h) for _ in range(world)]
    dist.all_gather(hs, h)
    agree = len({int(t.item()) for t in hs}) == 1

    # uncompressed NCCL allreduce on the same buffer size
    nccl_ms = None
    if args.nccl:
        y = x.clone()
        for _ in range(args.warmup):
            dist.all_reduce(y)
        nccl_ms = timed(lambda: dist.all_reduce(y), args.steps)

    # e2e through the C ABI with pinned host buffers: every step copies its
    # input host->device, allreduces, and copies its result device->host.
    # Steps are software-pipelined over three streams with two buffer sets
    # (PCIe is full duplex: step k's result read overlaps step k+1's input
    # copy and allreduce); every copy of every step is inside the region.
    (hx, hy0, hy1), numa_note = pinned_local(local, [(n, torch.float32)] * 3)
    hx.copy_(torch.from_numpy(x_host))
    hy = [hy0, hy1]
    dx = [torch.empty_like(x), x]  # x is free again (its checks are done)
    dout = [out, torch.empty_like(x)]
    s_in, s_ar, s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    ev_in = [torch.cuda.Event() for _ in range(2)]
    ev_ar = [torch.cuda.Event() for _ in range(2)]
    ev_out = [torch.cuda.Event() for _ in range(2)]
    for e in ev_ar + ev_out:
        e.record(torch.cuda.current_stream())
    e2e_steps = max(4, min(args.steps, 10))
    k_step = [0]

    def e2e_step():
        b = k_step[0] % 2
        k_step[0] += 1
        with torch.cuda.stream(s_in):
            s_in.wait_event(ev_ar[b])  # dx[b] free: step k-2's allreduce is done
            dx[b].copy_(hx, non_blocking=True)
            ev_in[b].record(s_in)
        with torch.cuda.stream(s_ar):
            s_ar.wait_event(ev_in[b])
            s_ar.wait_event(ev_out[b])  # dout[b] free: step k-2's result is read
            comm.allreduce(dx[b], spec, 0, dout[b])
            ev_ar[b].record(s_ar)
        with torch.cuda.stream(s_out):
            s_out.wait_event(ev_ar[b])
            hy[b].copy_(dout[b], non_blocking=True)
            ev_out[b].record(s_out)

    for _ in range(2):
        e2e_step()
    torch.cuda.synchronize()
    dist.barrier()
    w0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_step()
    torch.cuda.synchronize()
    e2e_s = torch.tensor([(time.perf_counter() - w0) / e2e_steps], device="cuda")
    dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
    e2e_s = float(e2e_s.item())

    cpu = None
    if rank == 0:
        # the reference's simulator on the full workload (all p ranks in one
        # process, as the reference is designed): p x n values, one call
        xs = np.stack([x_host] + [synth(1234 + j, n) for j in range(1, world)])
        sec, kind = cpu_allreduce(xs, rate, reps=1)
        del xs
        cpu = {"value": round(4 * n / sec / 1e9, 5), "unit": "GB/s",
               "cores": host_threads() if kind == "reference" else 1, "kind": kind,
               "sample": f"full workload: hcc::allreduce of {n} values per rank, p={world} ranks simulated in one "
                         f"process (the reference design), fixed-rate:{rate}, one call"}

    hbm, peak_src = peaks()
    W = wire_size_bytes(spec, c)
    p = world
    # per-rank algorithmic bytes of the fused kernel
    hbm_bytes = (p - 1) * (4 * c + 2 * W) + (4 * c + W) + p * (W + 4 * c)
    wire_bytes = 2 * (p - 1) * W
    t = ms * 1e-3
    hbm_ach = hbm_bytes / t / 1e9
    nvl_ach = wire_bytes / t / 1e9
    bound = "hbm" if hbm_bytes / (hbm * 1e9) >= wire_bytes / (NVLINK_PEAK * 1e9) else "nvlink"
    t_roof = max(hbm_bytes / (hbm * 1e9), wire_bytes / (NVLINK_PEAK * 1e9))
    if rank == 0:
        line = {
            "metric": METRIC, "value": round(4 * n / t / 1e9, 2), "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 5), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (hcc::Rng(1234+rank) 1e-3*normal() fp32 gradients, the reference's stream)",
            "config": workload_config(world, n, rate),
            "detail": {"l2": "inputs larger than L2 (256 MiB per rank)",
                       "engine": "one persistent fused kernel per rank, NVLink peer pushes (CUDA IPC)",
                       "wire_bytes_per_rank": wire_bytes,
                       "roofline_time_ms": round(t_roof * 1e3, 4),
                       "frac_of_roofline_time": round(t_roof / t, 4),
                       "soak": f"{soak} calls ({soak * soak_ms:.0f} ms) before the timed region, clocks sampled",
                       "soak_ms_per_call": round(soak_ms, 5),
                       "nccl_allreduce_GBps": round(4 * n / (nccl_ms * 1e-3) / 1e9, 2) if nccl_ms else None,
                       "nccl_ms": round(nccl_ms, 5) if nccl_ms else None,
                       "nccl_log": "profiles/r02_nccl_info_p*.txt (tools/nccl_info.py, NCCL_DEBUG=INFO)"},
            "parity": dict(parity, ranks_agree=agree),
            "roofline": {"bound": bound, "kernel": "ring_fused_kernel",
                         "achieved": round(hbm_ach if bound == "hbm" else nvl_ach, 1),
                         "peak": hbm if bound == "hbm" else NVLINK_PEAK, "unit": "GB/s",
                         "frac": round((hbm_ach / hbm) if bound == "hbm" else (nvl_ach / NVLINK_PEAK), 4),
                         "peak_source": peak_src if bound == "hbm" else "NVLink measured peer copy, B200_PROFILING.md",
                         "hbm_bytes_per_launch": hbm_bytes, "nvlink_bytes_per_launch": wire_bytes,
                         "hbm_frac": round(hbm_ach / hbm, 4), "nvlink_frac": round(nvl_ach / NVLINK_PEAK, 4),
                         "nvlink_frac_of_nominal_900": round(nvl_ach / NVLINK_NOMINAL, 4),
                         "traffic": traffic_for("ring_fused")},
            "cpu_baseline": cpu,
            "e2e": {"value": round(4 * n / e2e_s / 1e9, 3), "unit": "GB/s", "h2d_bytes_per_step": 4 * n,
                    "d2h_bytes_per_step": 4 * n, "api": "hccx_allreduce (C ABI) with pinned host in/out",
                    "pipeline": "steps overlapped over 3 streams x 2 buffer sets (H2D | allreduce | D2H)",
                    "host_buffers": numa_note,
                    "timer": "host wall clock, device synced both sides, max over ranks"},
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    ok = torch.tensor([1 if (rank != 0 or parity["bit_exact"]) and agree else 0], device="cuda")
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    comm.close()
    dist.destroy_process_group()
    if not int(ok.item()):
        sys.exit("bench: allreduce output differs from the CPU oracle or ranks disagree")


# ------------------------------------------------------- reference arm ----

def bench_reference(args):
    import numpy as np

    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    n_gpus = args.gpus
    rate = args.rate
    threads = host_threads()
    if n_gpus <= 1:
        n = args.n or (1 << 24)
        x = synth(1234, n)
        sample = f"full workload: {n} values, fixed-rate:{rate} compress+decompress (OpenMP, {threads} threads)"
        run = lambda: cpu_codec_roundtrip(n, rate, reps=1, x=x)  # noqa: E731
        warm = run
    else:
        p = n_gpus
        n = args.n or (1 << 26)
        n -= n % (64 * p)
        xs = np.stack([synth(1234 + j, n) for j in range(p)])
        ws = np.ascontiguousarray(xs[:, : (1 << 20) // (64 * p) * 64 * p])
        sample = (f"full workload per timed step: hcc::allreduce of {n} values per rank, p={p}, all ranks "
                  f"simulated in one process (reference design), fixed-rate:{rate}; warm-up steps on "
                  f"{ws.shape[1]} values per rank")
        run = lambda: cpu_allreduce(xs, rate, reps=1)  # noqa: E731
        warm = lambda: cpu_allreduce(ws, rate, reps=1)  # noqa: E731
    for _ in range(args.warmup):
        warm()
    ts = []
    kind = "port"
    for _ in range(args.steps):
        t, kind = run()
        ts.append(t)
    sec = sum(ts) / len(ts)
    value = round(4 * n / sec / 1e9, 5)
    line = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": n_gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(sec * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (hcc::Rng(1234+rank) 1e-3*normal() fp32 gradients, the reference's stream)",
        "config": workload_config(n_gpus, n, rate),
        "impl": "reference",
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": threads if kind == "reference" else 1,
                         "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _free_port() -> int:
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="hccx", choices=["hccx", "reference"])
    ap.add_argument("--rate", type=int, default=8)
    ap.add_argument("--n", type=int, default=0, help="values per rank (default: the BASELINE config size)")
    ap.add_argument("--nccl", type=int, default=1, help="also time an uncompressed NCCL allreduce (N>1)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        bench_reference(args)
        return
    world = int(os.environ.get("WORLD_SIZE", "0"))
    if args.gpus > 1 and world == 0:
        # not under torchrun: launch one rank per GPU ourselves
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", str(args.gpus),
               "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__)]
        sys.exit(subprocess.call(cmd + sys.argv[1:], env=dict(os.environ, OMP_NUM_THREADS=os.environ.get(
            "OMP_NUM_THREADS", str(host_threads())))))
    if world > 1:
        bench_allreduce(args)
    else:
        bench_codec(args)


if __name__ == "__main__":
    main()
