"""Experiment runner (the reference specifies it at
SPEC.md:362-413 but never built it): ``python -m paper_2409_02423_b200
{run,sweep,codec-bench,validate} --config PATH --out DIR``.

Config (JSON, or an INI-style ``[section] key = value`` file with the same
schema; values are JSON literals or bare strings):

  topology  {"preset": "b200-box" | "lassen-like" | "desk-2x2", "num_nodes": 1}
            or {"num_nodes": N, "gpus_per_node": G}; HYBRIDCOMM_PRESET overrides preset
  layout    {"dp": 2, "pp": 2, "tp": 2, "zero1": "off" | "replace" | "redundant"}
  model     ToyModelConfig fields (trainer.py)
  scheme    {"name": "z-hybrid:16,8"} or {"paths": {"DpAllReduce": "fixed-rate:4", ...}}
  seeds     [1, 2, ...] (default: model.seed)
  sweep     {"schemes": ["no-compression", "naive-zfp8", ...]}
  codec_bench {"sizes": [65536, ...], "codecs": ["identity", "fixed-rate:8", ...]}

run writes loss.csv, trace.csv and summary.json; sweep writes sweep.csv;
codec-bench writes codec_bench.csv.  An invalid config exits 2 with a
diagnostic naming the field; a diverged run exits 0 with "diverged": true.
Timing columns are measured device time (the reference's alpha-beta model is
replaced by measurement), so only they differ between identical runs.
"""
from __future__ import annotations

import argparse
import configparser
import csv
import io
import json
import os
import sys
from typing import Any, Dict, List

from .codec import CodecSpec, codec_spec_from_string, to_string
from .comm_path import CommPath, comm_path_from_string
from .errors import ConfigError, Error
from .netsim import Topology, write_trace_csv
from .parallel3d import SchemeTable, build_layout, scheme_from_name

SECTIONS = ("topology", "layout", "model", "scheme", "seeds", "sweep", "codec_bench")


def _literal(v: str) -> Any:
    try:
        return json.loads(v)
    except ValueError:
        return v


def parse_config(text: str) -> Dict[str, Any]:
    """JSON, or INI sections with JSON-literal values."""
    s = text.strip()
    if s.startswith("{"):
        try:
            cfg = json.loads(s)
        except ValueError as e:
            raise ConfigError("config", f"bad JSON: {e}") from None
    else:
        cp = configparser.ConfigParser()
        cp.optionxform = str
        try:
            cp.read_string(text)
        except configparser.Error as e:
            raise ConfigError("config", f"bad INI: {e}") from None
        cfg = {}
        for sec in cp.sections():
            items = {k: _literal(v) for k, v in cp.items(sec)}
            if sec == "seeds":
                cfg[sec] = items.get("list", list(items.values()))
            elif sec == "scheme" and "paths" not in items and any(k in CommPath.__members__ for k in items):
                cfg[sec] = {"paths": items}
            else:
                cfg[sec] = items
    if not isinstance(cfg, dict):
        raise ConfigError("config", "top level must be an object")
    for k in cfg:
        if k not in SECTIONS:
            raise ConfigError(k, "unknown section")
    return cfg


def serialize_config(cfg: Dict[str, Any]) -> str:
    return json.dumps(cfg, sort_keys=True, indent=1)


def make_topology(cfg: Dict[str, Any]) -> Topology:
    t = cfg.get("topology", {})
    preset = os.environ.get("HYBRIDCOMM_PRESET") or t.get("preset")
    if preset:
        topo = Topology.preset(preset, int(t.get("num_nodes", 1)))
        if "gpus_per_node" in t:
            topo.gpus_per_node = int(t["gpus_per_node"])
        return topo
    lay = cfg.get("layout", {})
    world = int(lay.get("dp", 1)) * int(lay.get("pp", 1)) * int(lay.get("tp", 1))
    # no preset: the given shape with one B200 box's link / codec / compute rates
    nn = int(t.get("num_nodes", 1))
    topo = Topology.b200_box(int(t.get("gpus_per_node", world)))
    topo.num_nodes = nn
    return topo


def make_scheme(cfg: Dict[str, Any], name: str = "") -> SchemeTable:
    sc = cfg.get("scheme", {"name": "no-compression"})
    if name:
        return scheme_from_name(name)
    if "paths" in sc:
        base = scheme_from_name(sc.get("name", "no-compression"))
        paths = dict(base.paths)
        for k, v in sc["paths"].items():
            paths[comm_path_from_string(k)] = codec_spec_from_string(str(v))
        return SchemeTable(sc.get("name", "custom"), paths)
    if "name" not in sc:
        raise ConfigError("scheme.name", "missing")
    return scheme_from_name(str(sc["name"]))


def make_trainer_inputs(cfg: Dict[str, Any]):
    from . import trainer as T

    topo = make_topology(cfg)
    lay = cfg.get("layout", {})
    for k in lay:
        if k not in ("dp", "pp", "tp", "zero1"):
            raise ConfigError(f"layout.{k}", "unknown field")
    try:
        layout = build_layout(int(lay.get("dp", 1)), int(lay.get("pp", 1)), int(lay.get("tp", 1)), topo.world_size())
    except Error as e:
        raise ConfigError("layout", str(e)) from None
    zero = T.zero_mode_from_string(str(lay.get("zero1", "off")))
    fields = T.ToyModelConfig.__dataclass_fields__
    model = cfg.get("model", {})
    for k in model:
        if k not in fields:
            raise ConfigError(f"model.{k}", "unknown field")
    mc = T.ToyModelConfig(**model)
    mc.validate(layout)
    return mc, layout, topo, zero


def validate(cfg: Dict[str, Any]) -> None:
    make_trainer_inputs(cfg)
    make_scheme(cfg)
    for s in cfg.get("sweep", {}).get("schemes", []):
        scheme_from_name(str(s))
    for c in cfg.get("codec_bench", {}).get("codecs", []):
        codec_spec_from_string(str(c))


def _run_one(cfg: Dict[str, Any], scheme: SchemeTable, seed: int):
    from . import trainer as T

    mc, layout, topo, zero = make_trainer_inputs(cfg)
    mc.seed = seed
    tr = T.Trainer3D(mc, layout, topo, scheme, zero)
    met = tr.run()
    return met, tr.clock.trace()


def cmd_run(cfg: Dict[str, Any], out: str) -> int:
    scheme = make_scheme(cfg)
    seeds = cfg.get("seeds") or [cfg.get("model", {}).get("seed", 1)]
    os.makedirs(out, exist_ok=True)
    summaries = []
    for seed in seeds:
        met, trace = _run_one(cfg, scheme, int(seed))
        tag = f"seed{seed}" if len(seeds) > 1 else ""
        with open(os.path.join(out, f"loss{tag}.csv"), "w", newline="") as fh:
            w = csv.writer(fh)
            w.writerow(["step", "loss"])
            for i, l in enumerate(met.step_loss):
                w.writerow([i, repr(float(l))])
        with open(os.path.join(out, f"trace{tag}.csv"), "w") as fh:
            write_trace_csv(fh, trace)
        summaries.append({
            "scheme": scheme.name, "seed": int(seed), "steps_completed": met.steps_completed,
            "diverged": bool(met.diverged), "final_eval_loss": float(met.final_eval_loss),
            "simulated_seconds": met.simulated_seconds, "samples_per_sec": met.samples_per_sec,
            "bytes_by_path": {str(p): {"raw": b.raw, "wire": b.wire} for p, b in sorted(met.bytes_by_path.items())},
            "scheme_paths": {str(p): to_string(scheme.at(p)) for p in CommPath},
        })
    with open(os.path.join(out, "summary.json"), "w") as fh:
        json.dump(summaries[0] if len(summaries) == 1 else summaries, fh, indent=1)
    return 0


def cmd_sweep(cfg: Dict[str, Any], out: str) -> int:
    names = cfg.get("sweep", {}).get("schemes") or [cfg.get("scheme", {}).get("name", "no-compression")]
    seeds = cfg.get("seeds") or [cfg.get("model", {}).get("seed", 1)]
    os.makedirs(out, exist_ok=True)
    rows = []
    for name in names:
        for seed in seeds:
            met, _ = _run_one(cfg, scheme_from_name(str(name)), int(seed))
            _, layout, _, _ = make_trainer_inputs(cfg)
            wire = sum(b.wire for b in met.bytes_by_path.values())
            raw = sum(b.raw for b in met.bytes_by_path.values())
            rows.append([name, seed, layout.world(), met.steps_completed, int(met.diverged),
                         repr(float(met.final_eval_loss)), repr(float(met.step_loss[-1])) if met.step_loss else "",
                         raw, wire, f"{met.samples_per_sec:.6g}"])
    with open(os.path.join(out, "sweep.csv"), "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["scheme", "seed", "world_size", "steps", "diverged", "final_loss", "last_step_loss", "raw_bytes",
                    "wire_bytes", "samples_per_sec_measured"])
        w.writerows(rows)
    return 0


def cmd_codec_bench(cfg: Dict[str, Any], out: str) -> int:
    """Ratio and throughput per codec on sparse (gradient-like) and dense
    (activation-like) buffers."""
    import numpy as np
    import torch

    from .codec import compress, decompress

    cb = cfg.get("codec_bench", {})
    sizes = [int(s) for s in cb.get("sizes", [1 << 20])]
    codecs = [str(c) for c in cb.get("codecs", ["identity", "lossless", "fixed-rate:8", "fixed-rate:16", "zfp-rate:8"])]
    os.makedirs(out, exist_ok=True)
    g = torch.Generator(device="cuda").manual_seed(0)
    rows = []
    for n in sizes:
        dense = torch.randn(n, device="cuda", generator=g)
        sparse = dense * (torch.rand(n, device="cuda", generator=g) < 0.1) * 1e-3
        for cname in codecs:
            spec = codec_spec_from_string(cname)
            for kind, x in (("sparse", sparse), ("dense", dense)):
                cbuf = compress(spec, x)
                torch.cuda.synchronize()
                ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
                ev[0].record()
                cbuf = compress(spec, x)
                ev[1].record()
                y = decompress(cbuf)
                ev[2].record()
                torch.cuda.synchronize()
                ratio = 4 * n / max(cbuf.payload_bytes(), 1)
                tc, td = ev[0].elapsed_time(ev[1]) * 1e-3, ev[1].elapsed_time(ev[2]) * 1e-3
                err = float((y - x).abs().max()) if spec.is_lossy() else 0.0
                rows.append([cname, kind, n, f"{ratio:.4f}", f"{4 * n / tc / 1e9:.3f}", f"{4 * n / td / 1e9:.3f}",
                             f"{err:.3g}"])
    with open(os.path.join(out, "codec_bench.csv"), "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["codec", "data", "n", "ratio", "compress_GBps", "decompress_GBps", "max_abs_err"])
        w.writerows(rows)
    return 0


def main(argv: List[str] = None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2409_02423_b200")
    ap.add_argument("command", choices=["run", "sweep", "codec-bench", "validate"])
    ap.add_argument("--config", required=False, default=None)
    ap.add_argument("--out", default="hcc_out")
    ap.add_argument("--seeds", default=None, help="comma-separated seed list (overrides the config)")
    a = ap.parse_args(argv)
    try:
        text = open(a.config).read() if a.config else "{}"
        cfg = parse_config(text)
        if a.seeds:
            cfg["seeds"] = [int(s) for s in a.seeds.split(",")]
        validate(cfg)
    except (ConfigError, Error, OSError, ValueError, TypeError) as e:
        field = getattr(e, "field", "config")
        print(f"error: invalid config ({field}): {e}", file=sys.stderr)
        return 2
    if a.command == "validate":
        print(serialize_config(cfg))
        return 0
    return {"run": cmd_run, "sweep": cmd_sweep, "codec-bench": cmd_codec_bench}[a.command](cfg, a.out)
