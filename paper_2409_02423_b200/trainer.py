"""3D-parallel toy trainer driving the B200 collectives.

Mirror of hcc::Trainer3D (proj/include/hcc/toymodel.hpp:89-160,
proj/src/toymodel.cpp:125-555): a stack of width->hidden->width tanh MLP
blocks learning a fixed random teacher, sharded over a dp x pp x tp layout,
GPipe schedule (all microbatch forwards, then backwards in reverse order),
Adam with optional ZeRO-1.  Every communication goes through this package's
collectives (single-device group path: all ranks' buffers on one GPU, the
reference's all-members-in-one-call semantics) with the scheme table's codec
per CommPath -- the call sites of toymodel.cpp:290-459.

The host arithmetic follows the reference's numeric contract exactly
(toymodel.hpp:89-102, linalg.cpp): matmuls accumulate k in ascending order
in fp32 without contraction, tanh is the C library's tanhf, Adam in the
reference's operation order, losses summed sequentially; initial weights and
batches come from std::mt19937_64 streams (rng.hpp) re-implemented here.
With bit-exact collectives the whole run -- step losses, final weights and
per-path byte accounting -- equals the reference trainer's bit for bit
(tests/test_trainer_gpu.py against fixtures produced by the reference,
tests/golden/trainer.npz).  Only ``simulated_seconds`` differs: collectives
advance the clock by their measured device time.
"""
from __future__ import annotations

import ctypes
import ctypes.util
import enum
import math
from dataclasses import dataclass, field
from typing import Dict, List, Optional

import numpy as np

from . import collectives as K
from .comm_path import CommPath
from .errors import BadLayoutError, ConfigError, NonFiniteInputError
from .netsim import SimClock, Topology
from .parallel3d import ParallelLayout, SchemeTable

_M64 = (1 << 64) - 1
f32 = np.float32


# ------------------------------------------------------------------ rng ----

class MT19937_64:
    """std::mt19937_64 (the C++ standard's bit-exact specification)."""

    _N, _M = 312, 156

    def __init__(self, seed: int):
        mt = [0] * self._N
        mt[0] = seed & _M64
        for i in range(1, self._N):
            mt[i] = (6364136223846793005 * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i) & _M64
        self._mt, self._i = mt, self._N

    def _twist(self) -> None:
        mt, N, M = self._mt, self._N, self._M
        for i in range(N):
            y = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % N] & 0x7FFFFFFF)
            v = mt[(i + M) % N] ^ (y >> 1)
            if y & 1:
                v ^= 0xB5026F5AA96619E9
            mt[i] = v
        self._i = 0

    def __call__(self) -> int:
        if self._i >= self._N:
            self._twist()
        y = self._mt[self._i]
        self._i += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & _M64


class Rng:
    """hcc::Rng (proj/include/hcc/rng.hpp:14-45): uniform() = (u64 >> 40) * 2^-24."""

    def __init__(self, seed: int):
        self._g = MT19937_64(seed)

    def uniform_array(self, n: int, lo: float, hi: float) -> np.ndarray:
        u = np.array([self._g() >> 40 for _ in range(n)], dtype=np.float64).astype(f32) * f32(2.0 ** -24)
        lo32, hi32 = f32(lo), f32(hi)
        return (lo32 + (hi32 - lo32) * u).astype(f32)


def mix_seed(seed: int, stream: int) -> int:
    """toymodel.cpp:10-15 (splitmix64 finaliser)."""
    z = (seed + 0x9E3779B97F4A7C15 * (stream + 1)) & _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


_STUDENT, _TEACHER, _EVAL, _BATCH_BASE = 5, 7, 0xEEEE, 0x100000000


# --------------------------------------------------------------- linalg ----

_libm = ctypes.CDLL(ctypes.util.find_library("m"))
_libm.tanhf.restype = ctypes.c_float
_libm.tanhf.argtypes = [ctypes.c_float]


def tanhf(x: np.ndarray) -> np.ndarray:
    """The C library's tanhf element by element (numpy's float32 tanh differs
    from it in the last ulp for ~40% of inputs)."""
    flat = x.reshape(-1)
    return np.fromiter((_libm.tanhf(float(v)) for v in flat), dtype=f32, count=flat.size).reshape(x.shape)


def mm_nt(a: np.ndarray, b: np.ndarray, m: int, k: int, n: int) -> np.ndarray:
    """c[i,j] = sum_k a[i,k] * b[j,k], k ascending, fp32 (linalg.cpp:16-24)."""
    a, b = a.reshape(m, k), b.reshape(n, k)
    c = np.zeros((m, n), f32)
    for kk in range(k):
        c = c + np.multiply.outer(a[:, kk], b[:, kk])
    return c


def mm_nn(a: np.ndarray, b: np.ndarray, m: int, k: int, n: int) -> np.ndarray:
    """c[i,j] = sum_k a[i,k] * b[k,j] (linalg.cpp:6-14)."""
    a, b = a.reshape(m, k), b.reshape(k, n)
    c = np.zeros((m, n), f32)
    for kk in range(k):
        c = c + np.multiply.outer(a[:, kk], b[kk, :])
    return c


def mm_tn(a: np.ndarray, b: np.ndarray, m: int, k: int, n: int) -> np.ndarray:
    """c[i,j] = sum_k a[k,i] * b[k,j] (linalg.cpp:26-34)."""
    a, b = a.reshape(k, m), b.reshape(k, n)
    c = np.zeros((m, n), f32)
    for kk in range(k):
        c = c + np.multiply.outer(a[kk, :], b[kk, :])
    return c


def sq_sum(d: np.ndarray) -> np.float32:
    """l += diff * diff over the buffer, sequential fp32."""
    sq = (d * d).astype(f32).reshape(-1)
    return np.add.accumulate(sq, dtype=f32)[-1] if sq.size else f32(0)


# ---------------------------------------------------------------- model ----

@dataclass
class ToyModelConfig:
    """toymodel.hpp:17-33."""

    num_blocks: int = 4
    hidden_dim: int = 64
    input_dim: int = 32
    batch_size: int = 16
    microbatches: int = 2
    steps: int = 100
    seed: int = 1
    learning_rate: float = 1.0e-3
    adam_beta1: float = 0.9
    adam_beta2: float = 0.95
    adam_epsilon: float = 1.0e-8
    eval_batch_size: int = 64

    def validate(self, layout: ParallelLayout) -> None:
        """toymodel.cpp:25-47."""
        checks = [("model.num_blocks", lambda: self.num_blocks >= 1, "must be >= 1"),
                  ("model.hidden_dim", lambda: self.hidden_dim >= 1, "must be >= 1"),
                  ("model.input_dim", lambda: self.input_dim >= 1, "must be >= 1"),
                  ("model.batch_size", lambda: self.batch_size >= 1, "must be >= 1"),
                  ("model.microbatches", lambda: self.microbatches >= 1, "must be >= 1"),
                  ("model.steps", lambda: self.steps >= 0, "must be >= 0"),
                  ("model.eval_batch_size", lambda: self.eval_batch_size >= 1, "must be >= 1"),
                  ("model.hidden_dim", lambda: self.hidden_dim % layout.tp == 0, "must be divisible by tp"),
                  ("model.input_dim", lambda: self.input_dim % layout.tp == 0, "must be divisible by tp"),
                  ("model.num_blocks", lambda: self.num_blocks % layout.pp == 0, "must be divisible by pp"),
                  ("model.batch_size", lambda: self.batch_size % (layout.dp * self.microbatches) == 0,
                   "must be divisible by dp * microbatches")]
        for fld, ok, msg in checks:  # in order, like the reference's early throws
            if not ok():
                raise ConfigError(fld, msg)


class ZeroMode(enum.IntEnum):
    """toymodel.hpp:35-42."""

    Off = 0
    Replace = 1
    Redundant = 2


def zero_mode_from_string(s: str) -> ZeroMode:
    m = {"off": ZeroMode.Off, "replace": ZeroMode.Replace, "redundant": ZeroMode.Redundant}
    if s not in m:
        raise ConfigError("layout.zero1", f"unknown mode '{s}' (expected off | replace | redundant)")
    return m[s]


@dataclass
class FullModel:
    """toymodel.hpp:44-56: w1 [blocks, hidden, width], w2 [blocks, width, hidden]."""

    num_blocks: int
    width: int
    hidden: int
    w1: np.ndarray
    w2: np.ndarray


def init_model(num_blocks: int, width: int, hidden: int, seed: int) -> FullModel:
    """toymodel.cpp:62-80."""
    rng = Rng(seed)
    s1 = f32(1.0) / np.sqrt(f32(width))
    s2 = f32(1.0) / np.sqrt(f32(hidden))
    w1 = np.empty((num_blocks, hidden, width), f32)
    w2 = np.empty((num_blocks, width, hidden), f32)
    for b in range(num_blocks):
        w1[b] = rng.uniform_array(hidden * width, -s1, s1).reshape(hidden, width)
        w2[b] = rng.uniform_array(width * hidden, -s2, s2).reshape(width, hidden)
    return FullModel(num_blocks, width, hidden, w1, w2)


def make_teacher(cfg: ToyModelConfig) -> FullModel:
    return init_model(cfg.num_blocks, cfg.input_dim, cfg.hidden_dim, mix_seed(cfg.seed, _TEACHER))


def make_student_init(cfg: ToyModelConfig) -> FullModel:
    return init_model(cfg.num_blocks, cfg.input_dim, cfg.hidden_dim, mix_seed(cfg.seed, _STUDENT))


def model_forward(model: FullModel, x: np.ndarray, batch: int) -> np.ndarray:
    """toymodel.cpp:92-107 (serial matmuls)."""
    cur = x.reshape(batch, model.width).astype(f32)
    for b in range(model.num_blocks):
        h = tanhf(mm_nt(cur, model.w1[b], batch, model.width, model.hidden))
        cur = mm_nt(h, model.w2[b], batch, model.hidden, model.width)
    return cur


def gen_step_batch(seed: int, step: int, batch: int, dim: int) -> np.ndarray:
    return Rng(mix_seed(seed, _BATCH_BASE + step)).uniform_array(batch * dim, -1.0, 1.0).reshape(batch, dim)


def gen_eval_batch(seed: int, batch: int, dim: int) -> np.ndarray:
    return Rng(mix_seed(seed, _EVAL)).uniform_array(batch * dim, -1.0, 1.0).reshape(batch, dim)


@dataclass
class PathBytes:
    raw: int = 0
    wire: int = 0


@dataclass
class RunMetrics:
    """toymodel.hpp:78-87."""

    step_loss: List[np.float32] = field(default_factory=list)
    final_eval_loss: np.float32 = f32(0)
    simulated_seconds: float = 0.0
    samples_per_sec: float = 0.0
    diverged: bool = False
    steps_completed: int = 0
    bytes_by_path: Dict[CommPath, PathBytes] = field(default_factory=dict)


class Trainer3D:
    """hcc::Trainer3D (toymodel.cpp:125-535) over the B200 collectives."""

    def __init__(self, cfg: ToyModelConfig, layout: ParallelLayout, topo: Topology, scheme: SchemeTable,
                 zero: ZeroMode):
        topo.validate()  # toymodel.cpp:128
        if layout.world() != topo.world_size():
            raise BadLayoutError("layout world does not match topology world")
        cfg.validate(layout)
        self.cfg, self.layout, self.scheme, self.zero = cfg, layout, scheme, ZeroMode(zero)
        self.clock = SimClock(topo)
        self.hs = cfg.hidden_dim // layout.tp
        self.bps = cfg.num_blocks // layout.pp
        self.mb_rows = cfg.batch_size // (layout.dp * cfg.microbatches)
        D = cfg.input_dim
        self.local_params = self.bps * 2 * D * self.hs
        self.padded_params = (self.local_params + layout.dp - 1) // layout.dp * layout.dp
        self.teacher = make_teacher(cfg)
        student = make_student_init(cfg)
        world = layout.world()
        self.flat = [np.zeros(self.local_params, f32) for _ in range(world)]
        self.grad = [np.zeros(self.local_params, f32) for _ in range(world)]
        mlen = self.local_params if self.zero == ZeroMode.Off else self.padded_params // layout.dp
        self.adam_m = [np.zeros(mlen, f32) for _ in range(world)]
        self.adam_v = [np.zeros(mlen, f32) for _ in range(world)]
        self.step_index = 0
        for d in range(layout.dp):
            for p in range(layout.pp):
                for t in range(layout.tp):
                    r = layout.rank_of(d, p, t)
                    for lb in range(self.bps):
                        g = p * self.bps + lb
                        self._w1(r, lb)[:] = student.w1[g, t * self.hs:(t + 1) * self.hs, :]
                        self._w2(r, lb)[:] = student.w2[g, :, t * self.hs:(t + 1) * self.hs]

    # flat layout per rank: local blocks in stage order, w1 slice then w2 slice
    def _w1(self, r: int, lb: int) -> np.ndarray:
        D, hs = self.cfg.input_dim, self.hs
        o = lb * 2 * D * hs
        return self.flat[r][o:o + hs * D].reshape(hs, D)

    def _w2(self, r: int, lb: int) -> np.ndarray:
        D, hs = self.cfg.input_dim, self.hs
        o = lb * 2 * D * hs + hs * D
        return self.flat[r][o:o + D * hs].reshape(D, hs)

    def _advance_compute(self, rank: int, flops: float) -> None:
        cf = self.clock.topology().compute_flops
        if cf > 0:
            self.clock.advance(rank, flops / cf)

    def _forward_block(self, r: int, lb: int, x: np.ndarray, rows: int):
        D, hs = self.cfg.input_dim, self.hs
        a = tanhf(mm_nt(x, self._w1(r, lb), rows, D, hs))
        y = mm_nt(a, self._w2(r, lb), rows, hs, D)
        self._advance_compute(r, 2.0 * rows * D * hs * 2)
        return y, (x, a)

    def _backward_block(self, r: int, lb: int, acts, dy: np.ndarray, rows: int) -> np.ndarray:
        D, hs = self.cfg.input_dim, self.hs
        x, a = acts
        w1, w2 = self._w1(r, lb), self._w2(r, lb)
        da = mm_nn(dy, w2, rows, D, hs)
        dh = (da * (f32(1.0) - a * a)).astype(f32)
        dw2 = mm_tn(dy, a, D, rows, hs)
        dw1 = mm_tn(dh, x, hs, rows, D)
        dx = mm_nn(dh, w1, rows, hs, D)
        o = lb * 2 * D * hs
        g = self.grad[r]
        g[o:o + hs * D] = g[o:o + hs * D] + dw1.reshape(-1)
        g[o + hs * D:o + 2 * hs * D] = g[o + hs * D:o + 2 * hs * D] + dw2.reshape(-1)
        self._advance_compute(r, 2.0 * (2.0 * rows * D * hs * 2))
        return dx

    def step(self) -> np.float32:
        """toymodel.cpp:239-371: GPipe forward, loss, reverse backward, optimizer."""
        L, cfg = self.layout, self.cfg
        dp, pp, tp, m, B, D = L.dp, L.pp, L.tp, cfg.microbatches, self.mb_rows, cfg.input_dim
        self.clock.set_step(self.step_index)
        full_x = gen_step_batch(cfg.seed, self.step_index, cfg.batch_size, D)
        rpr = cfg.batch_size // dp
        xin = [[full_x[d * rpr + mu * B:d * rpr + (mu + 1) * B] for mu in range(m)] for d in range(dp)]
        target = [[model_forward(self.teacher, xin[d][mu], B) for mu in range(m)] for d in range(dp)]
        acts = {}
        pend_f: Dict = {}
        pend_b: Dict = {}
        y_final = {}
        tp_spec, pp_spec = self.scheme.at(CommPath.TpAllReduce), self.scheme.at(CommPath.PpP2p)
        for mu in range(m):  # forward
            for s in range(pp):
                for d in range(dp):
                    comm = K.Communicator(L.tp_group(L.rank_of(d, s, 0)))
                    cur = [xin[d][mu] if s == 0 else pend_f.pop((d, t, mu)) for t in range(tp)]
                    for lb in range(self.bps):
                        parts = []
                        for t in range(tp):
                            r = L.rank_of(d, s, t)
                            y, acts[(r, mu, lb)] = self._forward_block(r, lb, cur[t], B)
                            parts.append(y.reshape(-1))
                        outs = K.allreduce(self.clock, comm, parts, tp_spec, CommPath.TpAllReduce, K.ReduceMode.Sum)
                        cur = [o.reshape(B, D) for o in outs]
                    if s < pp - 1:
                        for t in range(tp):
                            pend_f[(d, t, mu)] = K.p2p(self.clock, L.rank_of(d, s, t), L.rank_of(d, s + 1, t),
                                                       cur[t].reshape(-1), pp_spec, CommPath.PpP2p).reshape(B, D)
                    else:
                        y_final[(d, mu)] = cur[0]
        loss_scale = f32(1.0) / f32(B * D)
        step_loss = f32(0)
        for d in range(dp):
            acc = f32(0)
            for mu in range(m):
                acc = f32(acc + sq_sum(y_final[(d, mu)] - target[d][mu]) * loss_scale)
            step_loss = f32(step_loss + acc / f32(m))
        step_loss = f32(step_loss / f32(dp))
        for g in self.grad:
            g[:] = 0
        dy_scale = f32(2.0) / f32(B * D)
        for mu in reversed(range(m)):  # backward
            for s in reversed(range(pp)):
                for d in range(dp):
                    comm = K.Communicator(L.tp_group(L.rank_of(d, s, 0)))
                    if s == pp - 1:
                        dl = (dy_scale * (y_final[(d, mu)] - target[d][mu])).astype(f32)
                        dy = [dl for _ in range(tp)]
                    else:
                        dy = [pend_b.pop((d, t, mu)) for t in range(tp)]
                    for lb in reversed(range(self.bps)):
                        parts = []
                        for t in range(tp):
                            r = L.rank_of(d, s, t)
                            parts.append(self._backward_block(r, lb, acts[(r, mu, lb)], dy[t], B).reshape(-1))
                        outs = K.allreduce(self.clock, comm, parts, tp_spec, CommPath.TpAllReduce, K.ReduceMode.Sum)
                        dy = [o.reshape(B, D) for o in outs]
                    if s > 0:
                        for t in range(tp):
                            pend_b[(d, t, mu)] = K.p2p(self.clock, L.rank_of(d, s, t), L.rank_of(d, s - 1, t),
                                                       dy[t].reshape(-1), pp_spec, CommPath.PpP2p).reshape(B, D)
        inv_m = f32(1.0) / f32(m)
        for g in self.grad:
            g[:] = g * inv_m
        self._optimizer_phase()
        self.step_index += 1
        return step_loss

    def _adam_shard(self, r: int, grad: np.ndarray, offset: int, count: int) -> None:
        """toymodel.cpp:373-399, in the reference's operation order."""
        cfg = self.cfg
        b1, b2, lr, eps = f32(cfg.adam_beta1), f32(cfg.adam_beta2), f32(cfg.learning_rate), f32(cfg.adam_epsilon)
        t = self.step_index + 1
        c1 = f32(1.0 - math.pow(float(b1), t))
        c2 = f32(1.0 - math.pow(float(b2), t))
        n = max(0, min(count, self.local_params - offset))  # the padding tail carries no parameters
        if n == 0:
            return
        g = grad[:n].astype(f32)
        mm, vv, w = self.adam_m[r], self.adam_v[r], self.flat[r]
        mm[:n] = b1 * mm[:n] + (f32(1.0) - b1) * g
        vv[:n] = b2 * vv[:n] + (f32(1.0) - b2) * g * g
        mhat = mm[:n] / c1
        vhat = vv[:n] / c2
        w[offset:offset + n] = w[offset:offset + n] - lr * mhat / (np.sqrt(vhat) + eps)

    def _optimizer_phase(self) -> None:
        """toymodel.cpp:401-459."""
        L = self.layout
        dp = L.dp
        shard = self.padded_params // dp
        for p in range(L.pp):
            for t in range(L.tp):
                comm = K.Communicator([L.rank_of(d, p, t) for d in range(dp)])
                gpad = []
                for d in range(dp):
                    g = np.zeros(self.padded_params, f32)
                    g[:self.local_params] = self.grad[comm.ranks[d]]
                    gpad.append(g)
                if self.zero == ZeroMode.Off:
                    avg = K.allreduce(self.clock, comm, gpad, self.scheme.at(CommPath.DpAllReduce),
                                      CommPath.DpAllReduce, K.ReduceMode.Average)
                    for d in range(dp):
                        self._adam_shard(comm.ranks[d], avg[d], 0, self.local_params)
                    continue
                if self.zero == ZeroMode.Replace:
                    gs = K.ring_reduce_scatter(self.clock, comm, gpad, self.scheme.at(CommPath.Zero1ReduceScatter),
                                               CommPath.Zero1ReduceScatter)
                    grad_shards = [(s / f32(dp)).astype(f32) for s in gs]
                else:
                    avg = K.allreduce(self.clock, comm, gpad, self.scheme.at(CommPath.DpAllReduce),
                                      CommPath.DpAllReduce, K.ReduceMode.Average)
                    grad_shards = [avg[d][d * shard:(d + 1) * shard] for d in range(dp)]
                updated = []
                for d in range(dp):
                    r = comm.ranks[d]
                    self._adam_shard(r, grad_shards[d], d * shard, shard)
                    u = np.zeros(shard, f32)
                    lo, hi = d * shard, min((d + 1) * shard, self.local_params)
                    if hi > lo:
                        u[:hi - lo] = self.flat[r][lo:hi]
                    updated.append(u)
                gathered = K.ring_allgather(self.clock, comm, updated, self.scheme.at(CommPath.Zero1AllGather),
                                            CommPath.Zero1AllGather)
                for d in range(dp):
                    self.flat[comm.ranks[d]][:] = gathered[d][:self.local_params]

    def run(self) -> RunMetrics:
        """toymodel.cpp:461-498: divergence is recorded, not thrown."""
        met = RunMetrics()
        for _ in range(self.cfg.steps):
            try:
                with np.errstate(over="ignore", invalid="ignore"):  # divergence is data, as in the reference
                    loss = self.step()
            except NonFiniteInputError:
                met.diverged = True
                break
            met.step_loss.append(loss)
            met.steps_completed += 1
            if not np.isfinite(loss):
                met.diverged = True
                break
        met.simulated_seconds = self.clock.max_time()
        met.samples_per_sec = (met.steps_completed * self.cfg.batch_size / met.simulated_seconds
                               if met.simulated_seconds > 0 else 0.0)
        student = self.assemble_replica(0)
        ex = gen_eval_batch(self.cfg.seed, self.cfg.eval_batch_size, self.cfg.input_dim)
        want = model_forward(self.teacher, ex, self.cfg.eval_batch_size)
        with np.errstate(over="ignore", invalid="ignore"):
            got = model_forward(student, ex, self.cfg.eval_batch_size)
            met.final_eval_loss = f32(sq_sum(got - want) / f32(got.size))
        if not np.isfinite(met.final_eval_loss):
            met.diverged = True
        for e in self.clock.trace():
            pb = met.bytes_by_path.setdefault(e.path, PathBytes())
            pb.raw += e.raw_bytes
            pb.wire += e.wire_bytes
        return met

    def assemble_replica(self, d: int) -> FullModel:
        """toymodel.cpp:500-535."""
        cfg, L, hs = self.cfg, self.layout, self.hs
        w1 = np.zeros((cfg.num_blocks, cfg.hidden_dim, cfg.input_dim), f32)
        w2 = np.zeros((cfg.num_blocks, cfg.input_dim, cfg.hidden_dim), f32)
        for p in range(L.pp):
            for t in range(L.tp):
                r = L.rank_of(d, p, t)
                for lb in range(self.bps):
                    g = p * self.bps + lb
                    w1[g, t * hs:(t + 1) * hs, :] = self._w1(r, lb)
                    w2[g, :, t * hs:(t + 1) * hs] = self._w2(r, lb)
        return FullModel(cfg.num_blocks, cfg.input_dim, cfg.hidden_dim, w1, w2)


def run_experiment(cfg: ToyModelConfig, layout: ParallelLayout, topo: Topology, scheme: SchemeTable,
                   zero: ZeroMode, trace_out: Optional[list] = None) -> RunMetrics:
    """toymodel.cpp:537-545."""
    tr = Trainer3D(cfg, layout, topo, scheme, zero)
    met = tr.run()
    if trace_out is not None:
        trace_out.extend(tr.clock.trace())
    return met
