"""Strict run-config parser with the reference's schema (proj/src/config.cpp:105-224, README.md:181-207).

Unknown keys anywhere are rejected and errors name the key path (config.cpp:17-82). The one extension is the
transport backend: ``transport.backend`` accepts ``"b200"`` (config.cpp:176-178 allows inprocess|tcp) and an
optional top-level ``"b200"`` object carries the backend knobs (dtype, global_allreduce, gemm, data, ...).
``run_id = fnv1a64(canonical dump) ^ seed`` like config.cpp:222 (the dump is Python's canonical JSON, so ids are
stable within this implementation, not byte-identical to nlohmann's).
"""
from __future__ import annotations

import json
from dataclasses import dataclass, field
from typing import List

from ._native import ConfigError
from .executors import ALGORITHMS, B200Options, TrainConfig


@dataclass
class VerifyRun:
    algorithm: str = "sequential"
    n_workers: int = 1
    n_groups: int = 1


@dataclass
class RunConfig:
    train: TrainConfig
    transport_backend: str = "b200"
    endpoints: List[str] = field(default_factory=list)
    verify_tolerance: float = 1e-8
    verify_runs: List[VerifyRun] = field(default_factory=list)
    run_id: int = 0


class _Obj:
    def __init__(self, j, path):
        if not isinstance(j, dict):
            raise ConfigError(f"{path or 'config root'} must be a JSON object")
        self.j, self.path, self.seen = j, path, set()

    def kp(self, k):
        return k if not self.path else f"{self.path}.{k}"

    def has(self, k):
        return k in self.j

    def get(self, k, typ, default):
        self.seen.add(k)
        if k not in self.j:
            return default
        return _as(self.j[k], typ, self.kp(k))

    def req(self, k, typ):
        self.seen.add(k)
        if k not in self.j:
            raise ConfigError(f"missing required key {self.kp(k)}")
        return _as(self.j[k], typ, self.kp(k))

    def raw(self, k):
        self.seen.add(k)
        if k not in self.j:
            raise ConfigError(f"missing required key {self.kp(k)}")
        return self.j[k]

    def child(self, k):
        return _Obj(self.raw(k), self.kp(k))

    def reject_unknown(self):
        for k in self.j:
            if k not in self.seen:
                raise ConfigError(f"unknown key {self.kp(k)}")


def _as(v, typ, path):
    if typ is str:
        if not isinstance(v, str):
            raise ConfigError(f"{path} must be a string")
    elif typ is bool:
        if not isinstance(v, bool):
            raise ConfigError(f"{path} must be a boolean")
    elif typ is int:
        if isinstance(v, bool) or not isinstance(v, int):
            raise ConfigError(f"{path} must be an integer")
    else:
        if isinstance(v, bool) or not isinstance(v, (int, float)):
            raise ConfigError(f"{path} must be a number")
        v = float(v)
    return v


def _fnv1a64(s: str) -> int:
    h = 1469598103934665603
    for b in s.encode():
        h ^= b
        h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h


def parse_run_config(text: str) -> RunConfig:
    try:
        doc = json.loads(text)
    except json.JSONDecodeError as e:
        raise ConfigError(f"config is not valid JSON: {e}") from None
    root = _Obj(doc, "")
    t = TrainConfig()
    t.algorithm = root.req("algorithm", str)
    if t.algorithm not in ALGORITHMS:
        raise ConfigError(f"algorithm: expected sequential|csgd|lsgd, got '{t.algorithm}'")
    t.n_workers = root.get("n_workers", int, 1)
    t.n_groups = root.get("n_groups", int, 1)
    t.local_batch = root.get("local_batch", int, 64)
    t.epochs = root.get("epochs", int, 1)
    t.iterations = root.get("iterations", int, 0)
    t.seed = root.get("seed", int, 42)

    model = root.child("model")
    ls = model.raw("layer_sizes")
    if not isinstance(ls, list) or not ls:
        raise ConfigError("model.layer_sizes must be a nonempty array of integers")
    if any(isinstance(e, bool) or not isinstance(e, int) for e in ls):
        raise ConfigError("model.layer_sizes must contain only integers")
    t.layer_sizes = list(ls)
    if model.get("activation", str, "relu") != "relu":
        raise ConfigError("model.activation: only 'relu' is supported")
    model.reject_unknown()

    if root.has("data"):
        d = root.child("data")
        src = d.get("source", str, "synthetic")
        if src != "synthetic":
            # CSV ingestion (dataset.cpp:72-117) is outside the step's scope on this backend
            raise ConfigError(f"data.source: expected synthetic (csv is not supported by the b200 backend), got '{src}'")
        t.n_samples = d.get("n_samples", int, t.n_samples)
        t.n_features = d.get("n_features", int, t.n_features)
        t.n_classes = d.get("n_classes", int, t.n_classes)
        t.spread = d.get("spread", float, t.spread)
        d.get("path", str, "")
        d.reject_unknown()

    if root.has("optim"):
        o = root.child("optim")
        t.mode = o.get("mode", str, "momentum")
        if t.mode not in ("plain", "momentum"):
            raise ConfigError(f"optim.mode: expected plain|momentum, got '{t.mode}'")
        t.base_lr = o.get("base_lr", float, t.base_lr)
        t.momentum = o.get("momentum", float, t.momentum)
        t.weight_decay = o.get("weight_decay", float, t.weight_decay)
        t.warmup_epochs = o.get("warmup_epochs", float, t.warmup_epochs)
        t.decay_every_epochs = o.get("decay_every_epochs", int, t.decay_every_epochs)
        t.decay_factor = o.get("decay_factor", float, t.decay_factor)
        o.reject_unknown()

    out = RunConfig(train=t)
    if root.has("transport"):
        tr = root.child("transport")
        out.transport_backend = tr.get("backend", str, "b200")
        if out.transport_backend not in ("inprocess", "tcp", "b200"):
            raise ConfigError("transport.backend: expected inprocess|tcp|b200")
        if tr.has("endpoints"):
            eps = tr.raw("endpoints")
            if not isinstance(eps, list) or any(not isinstance(e, str) for e in eps):
                raise ConfigError("transport.endpoints must contain host:port strings")
            out.endpoints = list(eps)
        t.collective_timeout_s = tr.get("timeout_s", float, t.collective_timeout_s)
        tr.reject_unknown()

    if root.has("delays"):
        dl = root.child("delays")
        t.io_delay_s = dl.get("io_delay_ms", float, 0.0) / 1000.0
        t.global_link_delay_s = dl.get("global_link_delay_ms", float, 0.0) / 1000.0
        dl.reject_unknown()

    if root.has("verify"):
        v = root.child("verify")
        out.verify_tolerance = v.get("tolerance", float, 1e-8)
        if v.has("runs"):
            runs = v.raw("runs")
            if not isinstance(runs, list):
                raise ConfigError("verify.runs must be an array")
            for i, r in enumerate(runs):
                ro = _Obj(r, f"verify.runs[{i}]")
                vr = VerifyRun(ro.req("algorithm", str), ro.get("n_workers", int, 1), ro.get("n_groups", int, 1))
                if vr.algorithm not in ALGORITHMS:
                    raise ConfigError(f"algorithm: expected sequential|csgd|lsgd, got '{vr.algorithm}'")
                ro.reject_unknown()
                out.verify_runs.append(vr)
        v.reject_unknown()

    if root.has("b200"):
        b = root.child("b200")
        o = B200Options()
        o.dtype = b.get("dtype", str, o.dtype)
        o.n_devices = b.get("n_devices", int, o.n_devices)
        o.global_allreduce = b.get("global_allreduce", str, o.global_allreduce)
        o.gemm = b.get("gemm", str, o.gemm)
        o.data = b.get("data", str, o.data)
        o.model = b.get("model", str, o.model)
        o.record_phases = b.get("record_phases", bool, o.record_phases)
        o.csgd_nccl = b.get("csgd_nccl", bool, o.csgd_nccl)
        o.synthetic_params = b.get("synthetic_params", int, o.synthetic_params)
        b.reject_unknown()
        t.b200 = o

    root.reject_unknown()
    out.run_id = _fnv1a64(json.dumps(doc, sort_keys=True, separators=(",", ":"))) ^ (t.seed & 0xFFFFFFFFFFFFFFFF)
    return out


def load_run_config(path: str) -> RunConfig:
    try:
        with open(path) as f:
            text = f.read()
    except OSError:
        raise ConfigError(f"cannot open config file {path}") from None
    return parse_run_config(text)
