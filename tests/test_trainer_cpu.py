"""Trainer host arithmetic pinned on the CPU: trainer.py with its collectives
replaced by the CPU oracle (oracle/hcc_oracle.c, itself pinned to the
reference) must reproduce the reference trainer's runs bit for bit
(tests/golden/trainer.npz).  TEST INFRASTRUCTURE: the oracle stands in for
the GPU collectives only inside this test; tests/test_trainer_gpu.py runs the
same cases through libhccx."""
import os
import sys
import types

import numpy as np
import pytest

import oracle_lib as O

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "golden"))
from make_golden import SMALL_CFG, TRAIN_CASES  # noqa: E402

GOLD = os.path.join(os.path.dirname(__file__), "golden", "trainer.npz")
_KIND = {0: "identity", 1: "lossless", 2: "fixed-rate", 3: "zfp-rate"}


def _oracle_collectives():
    from paper_2409_02423_b200 import collectives as K
    from paper_2409_02423_b200.errors import NonFiniteInputError
    from paper_2409_02423_b200.netsim import CollectiveKind, TraceEvent

    def commit(clock, ranks, acct, path, kind, size):
        clock.sync_to_max(ranks)
        clock.record(TraceEvent(0, path, kind, size, acct[0], acct[1], 0.0, acct[2]))

    def call(fn, *a):
        try:
            return fn(*a)
        except RuntimeError as e:
            if "status 1" in str(e):
                raise NonFiniteInputError("non-finite") from None
            raise

    def allreduce(clock, comm, inputs, spec, path, mode):
        p = comm.size()
        if p == 1:
            return [np.array(inputs[0], np.float32)]
        out, acct = call(O.allreduce, np.stack(inputs), _KIND[int(spec.kind)], spec.rate_bits, int(mode) == 1)
        commit(clock, comm.ranks, acct, path, CollectiveKind.AllReduce, p)
        return list(out)

    def ring_reduce_scatter(clock, comm, inputs, spec, path):
        p = comm.size()
        if p == 1:
            return [np.array(inputs[0], np.float32)]
        out, acct = call(O.reduce_scatter, np.stack(inputs), _KIND[int(spec.kind)], spec.rate_bits)
        commit(clock, comm.ranks, acct, path, CollectiveKind.ReduceScatter, p)
        return list(out)

    def ring_allgather(clock, comm, shards, spec, path):
        p = comm.size()
        if p == 1:
            return [np.array(shards[0], np.float32)]
        out, acct = call(O.allgather, np.stack(shards), _KIND[int(spec.kind)], spec.rate_bits)
        commit(clock, comm.ranks, acct, path, CollectiveKind.AllGather, p)
        return list(out)

    def p2p(clock, src, dst, buf, spec, path):
        out, acct = call(O.p2p, np.asarray(buf, np.float32), _KIND[int(spec.kind)], spec.rate_bits)
        clock.sync_to_max([src, dst])
        clock.record(TraceEvent(0, path, CollectiveKind.P2P, 2, acct[0], acct[1], 0.0, acct[2]))
        return out

    return types.SimpleNamespace(Communicator=K.Communicator, ReduceMode=K.ReduceMode, allreduce=allreduce,
                                 ring_reduce_scatter=ring_reduce_scatter, ring_allgather=ring_allgather, p2p=p2p)


@pytest.mark.parametrize("case", TRAIN_CASES, ids=[c[0] for c in TRAIN_CASES])
def test_host_math_with_oracle_collectives(monkeypatch, case):
    from paper_2409_02423_b200 import build_layout, scheme_from_name
    from paper_2409_02423_b200 import trainer as T
    from paper_2409_02423_b200.comm_path import CommPath
    from paper_2409_02423_b200.netsim import Topology

    monkeypatch.setattr(T, "K", _oracle_collectives())
    name, over, dp, pp, tp, scheme, zero = case
    g = np.load(GOLD)
    cfg = T.ToyModelConfig(**dict(SMALL_CFG, **over))
    world = dp * pp * tp
    tr = T.Trainer3D(cfg, build_layout(dp, pp, tp, world), Topology.b200_box(world), scheme_from_name(scheme),
                     T.ZeroMode(zero))
    met = tr.run()
    assert met.steps_completed == int(g[f"{name}__steps_completed"])
    assert np.array(met.step_loss, np.float32).tobytes() == g[f"{name}__step_loss"].tobytes(), name
    if not met.diverged:
        m = tr.assemble_replica(0)
        assert m.w1.reshape(-1).tobytes() == g[f"{name}__w1"].tobytes()
        assert m.w2.reshape(-1).tobytes() == g[f"{name}__w2"].tobytes()
        assert np.float32(met.final_eval_loss).tobytes() == np.float32(g[f"{name}__final_eval_loss"]).tobytes()
        pb = g[f"{name}__path_bytes"]
        for path in CommPath:
            got = met.bytes_by_path.get(path)
            assert ((got.raw, got.wire) if got else (0, 0)) == (int(pb[2 * int(path)]), int(pb[2 * int(path) + 1]))
