"""Thin helpers that drive the C ABI (include/hccx.h) with torch device
memory, for the parity tests.  Everything computes in libhccx's kernels."""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from paper_2409_02423_b200 import _lib
from paper_2409_02423_b200.errors import check

KIND = {"identity": 0, "lossless": 1, "fixed-rate": 2, "zfp-rate": 3}


def codec(kind: str, rate: int = 0):
    return _lib.Codec(KIND[kind], rate)


def wire(kind: str, rate: int, n: int) -> int:
    out = C.c_uint64()
    check(_lib.hccx_wire_size_bytes(codec(kind, rate), n, C.byref(out)))
    return out.value


def dev(x: np.ndarray, offset: int = 0, dtype=torch.float32, device: int = 0):
    """Copy to cuda:<device>, optionally at an element offset inside a larger
    buffer (to exercise unaligned pointers)."""
    t = torch.zeros(x.size + offset + 8, dtype=dtype, device=f"cuda:{device}")
    v = t[offset:offset + x.size]
    if x.size:
        v.copy_(torch.from_numpy(np.ascontiguousarray(x)))
    return v


def stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def compress(kind: str, rate: int, x: np.ndarray, in_off: int = 0, out_off: int = 0):
    """-> (payload bytes as numpy, status of the error flag)."""
    n = x.size
    d_in = dev(x, in_off)
    w = wire(kind, rate, n)
    out = torch.zeros(w + out_off + 64, dtype=torch.uint8, device="cuda:0")
    o = out[out_off:out_off + w]
    err = torch.zeros(1, dtype=torch.int32, device="cuda:0")
    check(_lib.hccx_compress(codec(kind, rate), d_in.data_ptr() if n else None, n,
                             o.data_ptr() if w else None, err.data_ptr(), stream()))
    st = _lib.hccx_flag_status(err.data_ptr(), stream())
    return o.cpu().numpy(), st


def decompress(kind: str, rate: int, payload: np.ndarray, n: int, in_off: int = 0, out_off: int = 0):
    d_in = dev(payload, in_off, torch.uint8)
    out = torch.zeros(n + out_off + 8, dtype=torch.float32, device="cuda:0")
    o = out[out_off:out_off + n]
    check(_lib.hccx_decompress(codec(kind, rate), d_in.data_ptr() if payload.size else None, payload.size, n,
                               o.data_ptr() if n else None, stream()))
    torch.cuda.synchronize()
    return o.cpu().numpy()


class Group:
    def __init__(self, p: int):
        h = C.c_void_p()
        check(_lib.hccx_group_create(p, 0, C.byref(h)))
        self.h = h.value
        self.p = p

    def __del__(self):
        try:
            _lib.hccx_group_destroy(self.h)
        except Exception:
            pass

    def _run(self, fn, *args):
        st = fn(self.h, *args)
        if st == 0:
            st = _lib.hccx_group_status(self.h, stream())
        return st

    def allreduce(self, x: np.ndarray, kind: str, rate: int = 0, average: bool = False, inplace=False):
        ins = [dev(x[j]) for j in range(self.p)]
        outs = ins if inplace else [torch.full_like(t, float("nan")) for t in ins]
        a, _ka = _lib.ptr_array([t.data_ptr() for t in ins])
        b, _kb = _lib.ptr_array([t.data_ptr() for t in outs])
        st = self._run(_lib.hccx_group_allreduce, a, b, x.shape[1], codec(kind, rate), int(average), stream())
        return np.stack([t.cpu().numpy() for t in outs]), st

    def reduce_scatter(self, x: np.ndarray, kind: str, rate: int = 0):
        ins = [dev(x[j]) for j in range(self.p)]
        c = x.shape[1] // self.p
        outs = [torch.full((c,), float("nan"), device="cuda:0") for _ in range(self.p)]
        a, _ka = _lib.ptr_array([t.data_ptr() for t in ins])
        b, _kb = _lib.ptr_array([t.data_ptr() for t in outs])
        st = self._run(_lib.hccx_group_reduce_scatter, a, b, x.shape[1], codec(kind, rate), stream())
        return np.stack([t.cpu().numpy() for t in outs]), st

    def allgather(self, s: np.ndarray, kind: str, rate: int = 0):
        ins = [dev(s[j]) for j in range(self.p)]
        c = s.shape[1]
        outs = [torch.full((c * self.p,), float("nan"), device="cuda:0") for _ in range(self.p)]
        a, _ka = _lib.ptr_array([t.data_ptr() for t in ins])
        b, _kb = _lib.ptr_array([t.data_ptr() for t in outs])
        st = self._run(_lib.hccx_group_allgather, a, b, c, codec(kind, rate), stream())
        return np.stack([t.cpu().numpy() for t in outs]), st

    def broadcast(self, x: np.ndarray, root: int, kind: str, rate: int = 0):
        src = dev(x)
        outs = [torch.full((x.size,), float("nan"), device="cuda:0") for _ in range(self.p)]
        b, _kb = _lib.ptr_array([t.data_ptr() for t in outs])
        st = self._run(_lib.hccx_group_broadcast, root, src.data_ptr(), b, x.size, codec(kind, rate), stream())
        return np.stack([t.cpu().numpy() for t in outs]), st

    def p2p(self, x: np.ndarray, kind: str, rate: int = 0):
        src = dev(x)
        out = torch.full((x.size,), float("nan"), device="cuda:0")
        st = self._run(_lib.hccx_group_p2p, src.data_ptr(), out.data_ptr(), x.size, codec(kind, rate), stream())
        return out.cpu().numpy(), st


class MComm(Group):
    """Single-process communicator (hccx_mcomm_*): member j on devices[j].
    With every member on cuda:0 the members are virtual ranks of ONE
    cooperative launch of the NVLink engine's kernels (ring_fused_kernel /
    oneshot_allreduce_kernel device code), so a 1-GPU box runs the exact
    multi-GPU data path; with distinct devices the same kernels talk over
    NVLink (peer access)."""

    def __init__(self, p: int, max_n: int, devices=None):
        h = C.c_void_p()
        self.devices = list(devices or [0] * p)
        devs = (C.c_int * p)(*self.devices)
        check(_lib.hccx_mcomm_create(p, devs, max_n, C.byref(h)))
        self.h = h.value
        self.p = p

    def __del__(self):
        try:
            _lib.hccx_mcomm_destroy(self.h)
        except Exception:
            pass

    def _run(self, fn, *args):
        st = fn(self.h, *args)
        if st == 0:
            st = _lib.hccx_mcomm_status(self.h, None)
        return st

    def _nan(self, n, j):
        return torch.full((n,), float("nan"), device=f"cuda:{self.devices[j]}")

    def allreduce(self, x, kind, rate=0, average=False, inplace=False):
        return self._coll(_lib.hccx_mcomm_allreduce, x, x.shape[1], x.shape[1], inplace,
                          (codec(kind, rate), int(average)))

    def reduce_scatter(self, x, kind, rate=0):
        return self._coll(_lib.hccx_mcomm_reduce_scatter, x, x.shape[1] // self.p, x.shape[1], False,
                          (codec(kind, rate),))

    def allgather(self, s, kind, rate=0):
        return self._coll(_lib.hccx_mcomm_allgather, s, s.shape[1] * self.p, s.shape[1], False,
                          (codec(kind, rate),))

    def _coll(self, fn, x, out_n, n_arg, inplace, tail):
        ins = [dev(x[j], device=self.devices[j]) for j in range(self.p)]
        outs = ins if inplace else [self._nan(out_n, j) for j in range(self.p)]
        a, _ka = _lib.ptr_array([t.data_ptr() for t in ins])
        b, _kb = _lib.ptr_array([t.data_ptr() for t in outs])
        st = self._run(fn, a, b, n_arg, *tail, None)
        return np.stack([t.cpu().numpy() for t in outs]), st

    def broadcast(self, x, root, kind, rate=0):
        src = dev(x, device=self.devices[root])
        outs = [self._nan(x.size, j) for j in range(self.p)]
        b, _kb = _lib.ptr_array([t.data_ptr() for t in outs])
        st = self._run(_lib.hccx_mcomm_broadcast, root, src.data_ptr(), b, x.size, codec(kind, rate), None)
        return np.stack([t.cpu().numpy() for t in outs]), st

    def p2p(self, x, kind, rate=0, src=0, dst=1):
        s = dev(x, device=self.devices[src])
        out = self._nan(x.size, dst)
        st = self._run(_lib.hccx_mcomm_p2p, src, dst, s.data_ptr(), out.data_ptr(), x.size, codec(kind, rate), None)
        return out.cpu().numpy(), st
