"""3D-parallel toy trainer over the B200 collectives vs the
reference trainer itself.

tests/golden/trainer.npz holds hcc::Trainer3D runs of the UNMODIFIED
reference (oracle/_ref, tests/golden/make_golden.py): step losses, final eval
loss, the assembled replica-0 weights and raw/wire bytes per CommPath.  The
port drives every collective through libhccx on the GPU; with bit-exact
collectives and the reference's host numeric contract the runs agree bit for
bit.  Cases re-express proj/tests/test_toymodel.cpp (LosslessTransparency,
Zero1 modes, EventCensus, GradientCompressionDiscipline, Divergence,
Determinism).
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden", "trainer.npz")

import sys  # noqa: E402

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "golden"))
from make_golden import SMALL_CFG, TRAIN_CASES  # noqa: E402


def _run(over, dp, pp, tp, scheme, zero, trace=None):
    from paper_2409_02423_b200 import build_layout, scheme_from_name
    from paper_2409_02423_b200 import trainer as T
    from paper_2409_02423_b200.netsim import Topology

    cfg = T.ToyModelConfig(**dict(SMALL_CFG, **over))
    world = dp * pp * tp
    tr = T.Trainer3D(cfg, build_layout(dp, pp, tp, world), Topology.b200_box(world), scheme_from_name(scheme),
                     T.ZeroMode(zero))
    met = tr.run()
    if trace is not None:
        trace.extend(tr.clock.trace())
    return met, tr.assemble_replica(0)


@pytest.mark.parametrize("case", TRAIN_CASES, ids=[c[0] for c in TRAIN_CASES])
def test_matches_reference_trainer(cuda, case):
    from paper_2409_02423_b200.comm_path import CommPath

    name, over, dp, pp, tp, scheme, zero = case
    g = np.load(GOLD)
    met, model = _run(over, dp, pp, tp, scheme, zero)
    want = g[f"{name}__step_loss"]
    assert met.steps_completed == int(g[f"{name}__steps_completed"])
    assert bool(met.diverged) == bool(g[f"{name}__diverged"])
    assert np.array(met.step_loss, np.float32).tobytes() == want.tobytes(), name
    if not met.diverged:
        assert np.float32(met.final_eval_loss).tobytes() == np.float32(g[f"{name}__final_eval_loss"]).tobytes()
        assert model.w1.reshape(-1).tobytes() == g[f"{name}__w1"].tobytes(), name
        assert model.w2.reshape(-1).tobytes() == g[f"{name}__w2"].tobytes(), name
        pb = g[f"{name}__path_bytes"]
        for path in CommPath:
            got = met.bytes_by_path.get(path)
            raw, wire = (got.raw, got.wire) if got else (0, 0)
            assert (raw, wire) == (int(pb[2 * int(path)]), int(pb[2 * int(path) + 1])), (name, path)


def test_event_census_and_discipline(cuda):
    """test_toymodel.cpp:203-246."""
    from paper_2409_02423_b200 import scheme_from_name
    from paper_2409_02423_b200.comm_path import CommPath

    trace = []
    _run({"steps": 1}, 2, 2, 2, "no-compression", 0, trace)
    dp = pp = tp = 2
    m, blocks = SMALL_CFG["microbatches"], SMALL_CFG["num_blocks"]
    count = {p: sum(1 for e in trace if e.path == p) for p in CommPath}
    assert count[CommPath.PpP2p] == dp * tp * m * (pp - 1) * 2
    assert count[CommPath.TpAllReduce] == dp * blocks * m * 2
    assert count[CommPath.DpAllReduce] == pp * tp
    trace = []
    scheme = scheme_from_name("mz-hybrid:8")
    _run({"steps": 1}, 2, 2, 2, "mz-hybrid:8", 0, trace)
    lossy = [e for e in trace if scheme.at(e.path).is_lossy()]
    assert len(lossy) == 4 and all(e.path == CommPath.DpAllReduce for e in lossy)


def test_zero1_paths_and_determinism(cuda):
    """test_toymodel.cpp:156-201, :281-295."""
    from paper_2409_02423_b200.comm_path import CommPath

    for zero, rs, ag, ar in ((1, 1, 1, 0), (2, 0, 1, 1)):
        trace = []
        _run({"steps": 1}, 2, 1, 1, "no-compression", zero, trace)
        assert (sum(e.path == CommPath.Zero1ReduceScatter for e in trace),
                sum(e.path == CommPath.Zero1AllGather for e in trace),
                sum(e.path == CommPath.DpAllReduce for e in trace)) == (rs, ag, ar)
    trace = []
    _run({"steps": 2, "batch_size": 8}, 1, 1, 1, "no-compression", 1, trace)
    assert trace == []
    a, ma = _run({"steps": 3}, 2, 2, 2, "z-hybrid:16,8", 1)
    b, mb = _run({"steps": 3}, 2, 2, 2, "z-hybrid:16,8", 1)
    assert np.array(a.step_loss).tobytes() == np.array(b.step_loss).tobytes()
    assert ma.w1.tobytes() == mb.w1.tobytes() and ma.w2.tobytes() == mb.w2.tobytes()
