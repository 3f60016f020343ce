"""ctypes bindings for the CPU oracles (TEST INFRASTRUCTURE ONLY).

* ``orc``  -- oracle/_build/liborc.so, the C restatement of the reference
  (oracle/hcc_oracle.c).  Always available: built by oracle/build_ref.sh with
  gcc, here or on the GPU box.
* ``ref``  -- oracle/_ref/libhcc_ref.so, the unmodified reference library
  compiled from /root/reference (dev container only; the prebuilt .so travels
  with the gpurun snapshot).  ``ref`` is None when it is absent.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may use
this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORC_SO = os.path.join(ROOT, "oracle", "_build", "liborc.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libhcc_ref.so")

KIND = {"identity": 0, "lossless": 1, "fixed-rate": 2, "zfp-rate": 3}

_f = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_u8 = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_u64 = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")


def _build():
    subprocess.run(["bash", os.path.join(ROOT, "oracle", "build_ref.sh")], check=True)


def _load_orc():
    src = os.path.join(ROOT, "oracle", "hcc_oracle.c")
    if not os.path.exists(ORC_SO) or os.path.getmtime(ORC_SO) < os.path.getmtime(src):
        _build()
    lib = C.CDLL(ORC_SO)
    u64, i32 = C.c_uint64, C.c_int
    lib.orc_fill.argtypes = [u64, i32, u64, C.c_float, C.c_float, _f]
    lib.orc_wire_size.argtypes = [i32, i32, u64]
    lib.orc_wire_size.restype = u64
    lib.orc_fr_compress.argtypes = [i32, _f, u64, _u8]
    lib.orc_fr_decompress.argtypes = [i32, _u8, u64, _f]
    lib.orc_pred_size.argtypes = [_f, u64]
    lib.orc_pred_size.restype = u64
    lib.orc_pred_compress.argtypes = [_f, u64, _u8]
    lib.orc_pred_compress.restype = u64
    lib.orc_pred_decompress.argtypes = [_u8, u64, u64, _f]
    lib.orc_zfp_compress.argtypes = [i32, _f, u64, _u8]
    lib.orc_zfp_decompress.argtypes = [i32, _u8, u64, _f]
    lib.orc_codec_roundtrip.argtypes = [i32, i32, _f, u64, _f]
    lib.orc_reduce_scatter.argtypes = [i32, u64, _f, i32, i32, _f, _u64]
    lib.orc_allgather.argtypes = [i32, u64, _f, i32, i32, _f, _u64]
    lib.orc_allreduce.argtypes = [i32, u64, _f, i32, i32, i32, _f, _u64]
    lib.orc_p2p.argtypes = [u64, _f, i32, i32, _f, _u64]
    lib.orc_broadcast.argtypes = [i32, u64, _f, i32, i32, _f, _u64]
    lib.orc_block_bound.argtypes = [_f, u64, i32]
    lib.orc_block_bound.restype = C.c_double
    lib.orc_ring_fold.argtypes = [i32, u64, _f, _f]
    return lib


def _load_ref():
    if not os.path.exists(REF_SO):
        if os.path.isdir("/root/reference/proj/src"):
            _build()
        else:
            return None
    lib = C.CDLL(REF_SO)
    u64, i32 = C.c_uint64, C.c_int
    lib.ref_compress.argtypes = [i32, i32, i32, _f, u64, _u8, u64, C.POINTER(u64), C.POINTER(C.c_uint32)]
    lib.ref_decompress.argtypes = [i32, i32, i32, _u8, u64, u64, C.c_uint32, _f]
    lib.ref_wire_size.argtypes = [i32, i32, u64, C.POINTER(u64)]
    if hasattr(lib, "ref_time_codec"):
        lib.ref_time_codec.argtypes = [i32, i32, _f, u64, i32, C.POINTER(C.c_double)]
        lib.ref_time_allreduce.argtypes = [i32, u64, _f, i32, i32, i32, C.POINTER(C.c_double)]
    lib.ref_container.argtypes = [i32, i32, _f, u64, _u8, u64, C.POINTER(u64)]
    lib.ref_allreduce.argtypes = [i32, u64, _f, i32, i32, i32, _f, _u64]
    lib.ref_reduce_scatter.argtypes = [i32, u64, _f, i32, i32, _f, _u64]
    lib.ref_allgather.argtypes = [i32, u64, _f, i32, i32, _f, _u64]
    lib.ref_p2p.argtypes = [u64, _f, i32, i32, _f, _u64]
    lib.ref_fill.argtypes = [u64, i32, u64, C.c_float, C.c_float, _f]
    lib.ref_train.argtypes = [i32, i32, i32, i32, i32, i32, u64, C.c_float, i32, i32, i32, C.c_char_p, i32, _f,
                              C.POINTER(C.c_int), C.POINTER(C.c_float), C.POINTER(C.c_int), _f, _f, _u64]
    return lib


orc = _load_orc()
ref = _load_ref()


# ---------------------------------------------------------------- helpers --

def fill(seed: int, mode: str, n: int, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
    """Reference buffer generators (oracles.cpp:9-36) via the restated hcc::Rng."""
    m = {"bits": 0, "finite": 1, "uniform": 2, "sparse": 3, "normal": 4}[mode]
    out = np.empty(n, np.float32)
    orc.orc_fill(seed, m, n, lo, hi, out)
    return out


def wire_size(kind: str, rate: int, n: int) -> int:
    return int(orc.orc_wire_size(KIND[kind], rate, n))


def fr_compress(rate: int, x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, np.float32)
    out = np.zeros(max(wire_size("fixed-rate", rate, x.size), 1), np.uint8)
    st = orc.orc_fr_compress(rate, x, x.size, out)
    if st:
        raise FloatingPointError("non-finite input")
    return out[: wire_size("fixed-rate", rate, x.size)]


def fr_decompress(rate: int, payload: np.ndarray, n: int) -> np.ndarray:
    out = np.empty(max(n, 1), np.float32)
    p = np.ascontiguousarray(payload, np.uint8)
    if p.size == 0:
        p = np.zeros(1, np.uint8)
    orc.orc_fr_decompress(rate, p, n, out)
    return out[:n]


def zfp_compress(rate: int, x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, np.float32)
    w = wire_size("zfp-rate", rate, x.size)
    out = np.zeros(max(w, 1), np.uint8)
    if orc.orc_zfp_compress(rate, x if x.size else np.zeros(1, np.float32), x.size, out):
        raise FloatingPointError("non-finite input")
    return out[:w]


def zfp_decompress(rate: int, payload: np.ndarray, n: int) -> np.ndarray:
    out = np.empty(max(n, 1), np.float32)
    p = np.ascontiguousarray(payload, np.uint8)
    if p.size == 0:
        p = np.zeros(1, np.uint8)
    orc.orc_zfp_decompress(rate, p, n, out)
    return out[:n]


def pred_compress(x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, np.float32)
    xs = x if x.size else np.zeros(1, np.float32)
    sz = int(orc.orc_pred_size(xs, x.size))
    out = np.zeros(max(sz, 1), np.uint8)
    got = orc.orc_pred_compress(xs, x.size, out)
    assert got == sz
    return out[:sz]


def pred_decompress(payload: np.ndarray, n: int) -> np.ndarray:
    out = np.empty(max(n, 1), np.float32)
    p = np.ascontiguousarray(payload, np.uint8)
    st = orc.orc_pred_decompress(p if p.size else np.zeros(1, np.uint8), p.size, n, out)
    if st:
        raise ValueError("corrupt payload")
    return out[:n]


def _coll(fn, *args):
    acct = np.zeros(3, np.uint64)
    st = fn(*args, acct)
    return st, acct


def allreduce(inputs: np.ndarray, kind: str, rate: int = 0, average: bool = False):
    """inputs: [p, n] float32 -> ([p, n] outputs, (raw, wire, rounds))."""
    x = np.ascontiguousarray(inputs, np.float32)
    p, n = x.shape
    out = np.empty_like(x)
    st, acct = _coll(orc.orc_allreduce, p, n, x.reshape(-1), KIND[kind], rate, int(average), out.reshape(-1))
    if st:
        raise RuntimeError(f"oracle status {st}")
    return out, tuple(int(a) for a in acct)


def reduce_scatter(inputs: np.ndarray, kind: str, rate: int = 0):
    x = np.ascontiguousarray(inputs, np.float32)
    p, n = x.shape
    out = np.empty((p, n // p), np.float32)
    st, acct = _coll(orc.orc_reduce_scatter, p, n, x.reshape(-1), KIND[kind], rate, out.reshape(-1))
    if st:
        raise RuntimeError(f"oracle status {st}")
    return out, tuple(int(a) for a in acct)


def allgather(shards: np.ndarray, kind: str, rate: int = 0):
    x = np.ascontiguousarray(shards, np.float32)
    p, c = x.shape
    out = np.empty((p, p * c), np.float32)
    st, acct = _coll(orc.orc_allgather, p, c, x.reshape(-1), KIND[kind], rate, out.reshape(-1))
    if st:
        raise RuntimeError(f"oracle status {st}")
    return out, tuple(int(a) for a in acct)


def p2p(x: np.ndarray, kind: str, rate: int = 0):
    x = np.ascontiguousarray(x, np.float32)
    out = np.empty_like(x)
    st, acct = _coll(orc.orc_p2p, x.size, x if x.size else np.zeros(1, np.float32), KIND[kind], rate,
                     out if out.size else np.zeros(1, np.float32))
    if st:
        raise RuntimeError(f"oracle status {st}")
    return out, tuple(int(a) for a in acct)


def broadcast(x: np.ndarray, p: int, kind: str, rate: int = 0):
    x = np.ascontiguousarray(x, np.float32)
    out = np.empty((p, x.size), np.float32)
    st, acct = _coll(orc.orc_broadcast, p, x.size, x, KIND[kind], rate, out.reshape(-1))
    if st:
        raise RuntimeError(f"oracle status {st}")
    return out, tuple(int(a) for a in acct)


def block_bound(x: np.ndarray, rate: int) -> float:
    x = np.ascontiguousarray(x, np.float32)
    return float(orc.orc_block_bound(x, x.size, rate))


def ring_fold(inputs: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(inputs, np.float32)
    p, n = x.shape
    out = np.empty(n, np.float32)
    orc.orc_ring_fold(p, n, x.reshape(-1), out)
    return out


# ------------------------------------------------ the reference itself ----

def ref_compress(kind: str, rate: int, x: np.ndarray, serial: bool = False):
    x = np.ascontiguousarray(x, np.float32)
    cap = 4 * x.size + 4096 + (x.size // 4096 + 1) * 8
    out = np.zeros(cap, np.uint8)
    ln, cc = C.c_uint64(0), C.c_uint32(0)
    st = ref.ref_compress(KIND[kind], rate, int(serial), x if x.size else np.zeros(1, np.float32), x.size,
                          out, cap, C.byref(ln), C.byref(cc))
    if st:
        raise RuntimeError(f"reference status {st}")
    return out[: ln.value], cc.value


def ref_decompress(kind: str, rate: int, payload: np.ndarray, n: int, chunk_count: int, serial=False):
    out = np.empty(max(n, 1), np.float32)
    p = np.ascontiguousarray(payload, np.uint8)
    st = ref.ref_decompress(KIND[kind], rate, int(serial), p if p.size else np.zeros(1, np.uint8), p.size, n,
                            chunk_count, out)
    if st:
        raise RuntimeError(f"reference status {st}")
    return out[:n]


def ref_fill(seed: int, mode: str, n: int, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
    m = {"bits": 0, "finite": 1, "uniform": 2, "sparse": 3}[mode]
    out = np.empty(max(n, 1), np.float32)
    ref.ref_fill(seed, m, n, lo, hi, out)
    return out[:n]


def ref_allreduce(inputs: np.ndarray, kind: str, rate: int = 0, average: bool = False):
    x = np.ascontiguousarray(inputs, np.float32)
    p, n = x.shape
    out = np.empty_like(x)
    acct = np.zeros(3, np.uint64)
    st = ref.ref_allreduce(p, n, x.reshape(-1), KIND[kind], rate, int(average), out.reshape(-1), acct)
    if st:
        raise RuntimeError(f"reference status {st}")
    return out, tuple(int(a) for a in acct)


def ref_reduce_scatter(inputs: np.ndarray, kind: str, rate: int = 0):
    x = np.ascontiguousarray(inputs, np.float32)
    p, n = x.shape
    out = np.empty((p, n // p), np.float32)
    acct = np.zeros(3, np.uint64)
    st = ref.ref_reduce_scatter(p, n, x.reshape(-1), KIND[kind], rate, out.reshape(-1), acct)
    if st:
        raise RuntimeError(f"reference status {st}")
    return out, tuple(int(a) for a in acct)


def ref_allgather(shards: np.ndarray, kind: str, rate: int = 0):
    x = np.ascontiguousarray(shards, np.float32)
    p, c = x.shape
    out = np.empty((p, p * c), np.float32)
    acct = np.zeros(3, np.uint64)
    st = ref.ref_allgather(p, c, x.reshape(-1), KIND[kind], rate, out.reshape(-1), acct)
    if st:
        raise RuntimeError(f"reference status {st}")
    return out, tuple(int(a) for a in acct)


def ref_p2p(x: np.ndarray, kind: str, rate: int = 0):
    x = np.ascontiguousarray(x, np.float32)
    out = np.empty(max(x.size, 1), np.float32)
    acct = np.zeros(3, np.uint64)
    st = ref.ref_p2p(x.size, x if x.size else np.zeros(1, np.float32), KIND[kind], rate, out, acct)
    if st:
        raise RuntimeError(f"reference status {st}")
    return out[: x.size], tuple(int(a) for a in acct)


def ref_train(cfg: dict, dp: int, pp: int, tp: int, scheme: str, zero: int):
    """hcc::Trainer3D::run via oracle/_ref (the reference compiled): returns a
    dict of step losses, final eval loss, replica-0 model and path bytes."""
    steps = cfg["steps"]
    nb, hid, w = cfg["num_blocks"], cfg["hidden_dim"], cfg["input_dim"]
    loss = np.zeros(max(steps, 1), np.float32)
    w1 = np.zeros(nb * hid * w, np.float32)
    w2 = np.zeros(nb * w * hid, np.float32)
    pb = np.zeros(12, np.uint64)
    done, ev, div = C.c_int(0), C.c_float(0), C.c_int(0)
    st = ref.ref_train(nb, hid, w, cfg["batch_size"], cfg["microbatches"], steps, cfg["seed"], cfg["learning_rate"],
                       dp, pp, tp, scheme.encode(), zero, loss, C.byref(done), C.byref(ev), C.byref(div), w1, w2, pb)
    if st:
        raise RuntimeError(f"reference status {st}")
    return {"step_loss": loss[: done.value], "steps_completed": done.value, "final_eval_loss": np.float32(ev.value),
            "diverged": bool(div.value), "w1": w1, "w2": w2, "path_bytes": pb}


def ref_time_codec(kind: str, rate: int, x: np.ndarray, reps: int = 1) -> float:
    """Median seconds of hcc::compress + hcc::decompress on the reference
    library itself (marshalling outside the timed region)."""
    x = np.ascontiguousarray(x, np.float32)
    s = C.c_double(0)
    st = ref.ref_time_codec(KIND[kind], rate, x, x.size, reps, C.byref(s))
    if st:
        raise RuntimeError(f"reference status {st}")
    return float(s.value)


def ref_time_allreduce(inputs: np.ndarray, kind: str, rate: int = 0, reps: int = 1) -> float:
    """Median seconds of hcc::allreduce (Sum) on the reference library."""
    x = np.ascontiguousarray(inputs, np.float32)
    p, n = x.shape
    s = C.c_double(0)
    st = ref.ref_time_allreduce(p, n, x.reshape(-1), KIND[kind], rate, reps, C.byref(s))
    if st:
        raise RuntimeError(f"reference status {st}")
    return float(s.value)
