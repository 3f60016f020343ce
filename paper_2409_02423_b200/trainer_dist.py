"""Trainer3D across processes: one GPU per rank, NVLink collectives.

The SPMD form of trainer.Trainer3D (proj/src/toymodel.cpp:239-459): every
process owns ONE rank's parameter shard, optimizer state and activations,
walks the reference's schedule (GPipe forwards, reverse-order backwards,
optimizer per DP group) in the same order as every other process, and
joins the collectives of its own TP group, PP chain and DP group through
hybrid.HybridComm (fused NVLink kernels, scheme per CommPath).  Host
arithmetic is trainer.py's (the reference's numeric contract) and the
collectives are bit-exact, so a run reproduces hcc::Trainer3D bit for bit:
step losses, the assembled replica-0 weights, the eval loss and the per-path
byte totals (tests/trainer_dist_parity.py against tests/golden/trainer.npz).

Launch under torchrun with world = dp * pp * tp; rank r plays layout rank r.
"""
from __future__ import annotations

import math
from typing import Dict, List

import numpy as np

from . import trainer as T
from .comm_path import CommPath
from .errors import NonFiniteInputError
from .parallel3d import ParallelLayout, SchemeTable

f32 = np.float32


class DistTrainer3D:
    def __init__(self, cfg: T.ToyModelConfig, layout: ParallelLayout, scheme: SchemeTable, zero: T.ZeroMode):
        import torch.distributed as dist

        from .hybrid import HybridComm

        cfg.validate(layout)
        self.cfg, self.layout, self.scheme, self.zero = cfg, layout, scheme, T.ZeroMode(zero)
        self.rank = dist.get_rank()
        c = layout.coord_of(self.rank)
        self.d, self.s, self.t = c.d, c.p, c.t
        self.hs = cfg.hidden_dim // layout.tp
        self.bps = cfg.num_blocks // layout.pp
        self.B = cfg.batch_size // (layout.dp * cfg.microbatches)
        D = cfg.input_dim
        self.local_params = self.bps * 2 * D * self.hs
        self.padded_params = (self.local_params + layout.dp - 1) // layout.dp * layout.dp
        self.teacher = T.make_teacher(cfg)
        student = T.make_student_init(cfg)
        self.flat = np.zeros(self.local_params, f32)
        for lb in range(self.bps):
            g = self.s * self.bps + lb
            self._w1(lb)[:] = student.w1[g, self.t * self.hs:(self.t + 1) * self.hs, :]
            self._w2(lb)[:] = student.w2[g, :, self.t * self.hs:(self.t + 1) * self.hs]
        self.grad = np.zeros(self.local_params, f32)
        mlen = self.local_params if self.zero == T.ZeroMode.Off else self.padded_params // layout.dp
        self.adam_m = np.zeros(mlen, f32)
        self.adam_v = np.zeros(mlen, f32)
        self.step_index = 0
        self.hc = HybridComm(layout, scheme, max(self.padded_params, self.B * D) + layout.world())
        self.bytes: Dict[CommPath, List[int]] = {p: [0, 0] for p in CommPath}

    # ------------------------------------------------------------ helpers
    def _w1(self, lb):
        D, hs = self.cfg.input_dim, self.hs
        o = lb * 2 * D * hs
        return self.flat[o:o + hs * D].reshape(hs, D)

    def _w2(self, lb):
        D, hs = self.cfg.input_dim, self.hs
        o = lb * 2 * D * hs + hs * D
        return self.flat[o:o + D * hs].reshape(D, hs)

    @staticmethod
    def _dev(x: np.ndarray):
        import torch

        return torch.from_numpy(np.ascontiguousarray(x, f32).reshape(-1)).cuda()

    def _tally(self, leader: bool) -> None:
        """Count a collective once (the reference records one event per
        call): the group's first rank, or the p2p source."""
        last = self.hc.last_bytes() if leader else None
        if last:
            path, raw, wire = last
            self.bytes[path][0] += raw
            self.bytes[path][1] += wire

    def _tp_allreduce(self, y: np.ndarray) -> np.ndarray:
        out = self.hc.tp_allreduce(self._dev(y))
        self._tally(self.layout.tp > 1 and self.t == 0)
        return out.cpu().numpy().reshape(y.shape)

    def _p2p(self, x: np.ndarray, src: int, dst: int) -> np.ndarray:
        out = self.hc.pp_send_recv(self._dev(x), src, dst)
        self._tally(self.s == src)
        return out.cpu().numpy().reshape(self.B, self.cfg.input_dim) if self.s == dst else None

    # --------------------------------------------------------------- step
    def step(self) -> np.float32:
        import torch
        import torch.distributed as dist

        cfg, L = self.cfg, self.layout
        dp, pp, m, B, D, hs = L.dp, L.pp, cfg.microbatches, self.B, cfg.input_dim, self.hs
        self.hc.step = self.step_index
        full_x = T.gen_step_batch(cfg.seed, self.step_index, cfg.batch_size, D)
        rpr = cfg.batch_size // dp
        xin = [full_x[self.d * rpr + mu * B:self.d * rpr + (mu + 1) * B] for mu in range(m)]
        acts, pend_f, pend_b, y_final = {}, {}, {}, {}
        for mu in range(m):  # forward (reference loop order; this rank acts on its own (d, s))
            for s in range(pp):
                if s == self.s:
                    cur = xin[mu] if s == 0 else pend_f.pop(mu)
                    for lb in range(self.bps):
                        a = T.tanhf(T.mm_nt(cur, self._w1(lb), B, D, hs))
                        acts[(mu, lb)] = (cur, a)
                        cur = self._tp_allreduce(T.mm_nt(a, self._w2(lb), B, hs, D))
                    if s < pp - 1:
                        self._p2p(cur, s, s + 1)
                    else:
                        y_final[mu] = cur
                elif s + 1 == self.s:
                    pend_f[mu] = self._p2p(np.zeros((B, D), f32), s, s + 1)
        # loss: replica d's last stage (t = 0) holds it; combined in replica order
        acc = f32(0)
        if self.s == pp - 1 and self.t == 0:
            scale = f32(1.0) / f32(B * D)
            for mu in range(m):
                tgt = T.model_forward(self.teacher, xin[mu], B)
                acc = f32(acc + T.sq_sum(y_final[mu] - tgt) * scale)
        torch.cuda.synchronize()  # no fused kernel in flight across an NCCL call
        accs = [torch.zeros(1, dtype=torch.float32, device="cuda") for _ in range(L.world())]
        dist.all_gather(accs, torch.tensor([float(acc)], dtype=torch.float32, device="cuda"))
        step_loss = f32(0)
        for d in range(dp):
            step_loss = f32(step_loss + f32(accs[L.rank_of(d, pp - 1, 0)].item()) / f32(m))
        step_loss = f32(step_loss / f32(dp))
        self.grad[:] = 0
        dy_scale = f32(2.0) / f32(B * D)
        for mu in reversed(range(m)):  # backward
            for s in reversed(range(pp)):
                if s == self.s:
                    if s == pp - 1:
                        dy = (dy_scale * (y_final[mu] - T.model_forward(self.teacher, xin[mu], B))).astype(f32)
                    else:
                        dy = pend_b.pop(mu)
                    for lb in reversed(range(self.bps)):
                        x, a = acts[(mu, lb)]
                        da = T.mm_nn(dy, self._w2(lb), B, D, hs)
                        dh = (da * (f32(1.0) - a * a)).astype(f32)
                        dw2 = T.mm_tn(dy, a, D, B, hs)
                        dw1 = T.mm_tn(dh, x, hs, B, D)
                        dx = T.mm_nn(dh, self._w1(lb), B, hs, D)
                        o = lb * 2 * D * hs
                        self.grad[o:o + hs * D] = self.grad[o:o + hs * D] + dw1.reshape(-1)
                        self.grad[o + hs * D:o + 2 * hs * D] = self.grad[o + hs * D:o + 2 * hs * D] + dw2.reshape(-1)
                        dy = self._tp_allreduce(dx)
                    if s > 0:
                        self._p2p(dy, s, s - 1)
                elif s - 1 == self.s:
                    pend_b[mu] = self._p2p(np.zeros((B, D), f32), s, s - 1)
        self.grad[:] = self.grad * (f32(1.0) / f32(m))
        self._optimizer_phase()
        self.step_index += 1
        return step_loss

    def _adam(self, grad: np.ndarray, offset: int, count: int) -> None:
        cfg = self.cfg
        b1, b2, lr, eps = f32(cfg.adam_beta1), f32(cfg.adam_beta2), f32(cfg.learning_rate), f32(cfg.adam_epsilon)
        t = self.step_index + 1
        c1 = f32(1.0 - math.pow(float(b1), t))
        c2 = f32(1.0 - math.pow(float(b2), t))
        n = max(0, min(count, self.local_params - offset))
        if n == 0:
            return
        g = grad[:n].astype(f32)
        mm, vv, w = self.adam_m, self.adam_v, self.flat
        mm[:n] = b1 * mm[:n] + (f32(1.0) - b1) * g
        vv[:n] = b2 * vv[:n] + (f32(1.0) - b2) * g * g
        w[offset:offset + n] = w[offset:offset + n] - lr * (mm[:n] / c1) / (np.sqrt(vv[:n] / c2) + eps)

    def _optimizer_phase(self) -> None:
        dp = self.layout.dp
        shard = self.padded_params // dp
        gpad = np.zeros(self.padded_params, f32)
        gpad[:self.local_params] = self.grad
        lead = dp > 1 and self.d == 0
        if self.zero == T.ZeroMode.Off:
            avg = self.hc.dp_allreduce(self._dev(gpad)).cpu().numpy()
            self._tally(lead)
            self._adam(avg, 0, self.local_params)
            return
        if self.zero == T.ZeroMode.Replace:
            gs = self.hc.zero_reduce_scatter(self._dev(gpad)).cpu().numpy()
            self._tally(lead)
            mine = (gs / f32(dp)).astype(f32)
        else:
            avg = self.hc.dp_allreduce(self._dev(gpad)).cpu().numpy()
            self._tally(lead)
            mine = avg[self.d * shard:(self.d + 1) * shard]
        self._adam(mine, self.d * shard, shard)
        upd = np.zeros(shard, f32)
        lo, hi = self.d * shard, min((self.d + 1) * shard, self.local_params)
        if hi > lo:
            upd[:hi - lo] = self.flat[lo:hi]
        full = self.hc.zero_allgather(self._dev(upd)).cpu().numpy()
        self._tally(lead)
        self.flat[:] = full[:self.local_params]

    # ---------------------------------------------------------------- run
    def run(self) -> T.RunMetrics:
        """Rank 0 returns the metrics (step losses, eval loss, path bytes);
        divergence is agreed across ranks and recorded, not thrown."""
        import torch
        import torch.distributed as dist

        met = T.RunMetrics()
        for _ in range(self.cfg.steps):
            bad = 0
            loss = f32(0)
            try:
                with np.errstate(over="ignore", invalid="ignore"):
                    loss = self.step()
                self.hc.status()
            except NonFiniteInputError:
                bad = 1
            torch.cuda.synchronize()
            flag = torch.tensor([bad], device="cuda")
            dist.all_reduce(flag)
            if flag.item():
                met.diverged = True
                break
            met.step_loss.append(loss)
            met.steps_completed += 1
            if not np.isfinite(loss):
                met.diverged = True
                break
        # assemble replica 0 on every rank (all_gather of the flat shards)
        torch.cuda.synchronize()
        flats = [torch.zeros(self.local_params, dtype=torch.float32, device="cuda") for _ in range(self.layout.world())]
        dist.all_gather(flats, torch.from_numpy(self.flat).cuda())
        self.replica0 = self._assemble([f.cpu().numpy() for f in flats], 0)
        ex = T.gen_eval_batch(self.cfg.seed, self.cfg.eval_batch_size, self.cfg.input_dim)
        with np.errstate(over="ignore", invalid="ignore"):
            want = T.model_forward(self.teacher, ex, self.cfg.eval_batch_size)
            got = T.model_forward(self.replica0, ex, self.cfg.eval_batch_size)
            met.final_eval_loss = f32(T.sq_sum(got - want) / f32(got.size))
        if not np.isfinite(met.final_eval_loss):
            met.diverged = True
        tallies = torch.tensor([v for p in CommPath for v in self.bytes[p]], dtype=torch.int64, device="cuda")
        dist.all_reduce(tallies)
        tl = tallies.tolist()
        for i, p in enumerate(CommPath):
            if tl[2 * i] or tl[2 * i + 1]:
                met.bytes_by_path[p] = T.PathBytes(tl[2 * i], tl[2 * i + 1])
        return met

    def _assemble(self, flats: List[np.ndarray], d: int) -> T.FullModel:
        cfg, L, hs, D = self.cfg, self.layout, self.hs, self.cfg.input_dim
        w1 = np.zeros((cfg.num_blocks, cfg.hidden_dim, D), f32)
        w2 = np.zeros((cfg.num_blocks, D, cfg.hidden_dim), f32)
        for p in range(L.pp):
            for t in range(L.tp):
                fl = flats[L.rank_of(d, p, t)]
                for lb in range(self.bps):
                    g = p * self.bps + lb
                    o = lb * 2 * D * hs
                    w1[g, t * hs:(t + 1) * hs, :] = fl[o:o + hs * D].reshape(hs, D)
                    w2[g, :, t * hs:(t + 1) * hs] = fl[o + hs * D:o + 2 * hs * D].reshape(D, hs)
        return T.FullModel(cfg.num_blocks, D, cfg.hidden_dim, w1, w2)

    def close(self) -> None:
        self.hc.close()
