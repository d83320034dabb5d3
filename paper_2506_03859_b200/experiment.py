"""The reference's experiment driver on the B200 engine: the caller of the QB path.

Mirrors rsvd::ExperimentConfig / run_experiment / execute_run and the three report
files (/root/reference/proj/include/rsvd/experiment.hpp:16-88,
/root/reference/proj/src/experiment.cpp):

    load_experiment_config(path)  JSON config, same keys, defaults and validation
                                  messages (experiment.cpp:59-78, 262-304)
    build_grid(cfg)               algorithms x targets x power x density x trials,
                                  seed = cfg.seed + 0x9E3779B97F4A7C15 (i + 1) (:80-107)
    execute_run(...)              one fixed-precision or fixed-rank run, timed, then
                                  truncate_to_tolerance and the exact relative error
                                  (:114-169) -- all on the GPU
    aggregate(records, runs)      per-cell means in first-occurrence order (:171-214)
    write_report_csv / read_report_csv / write_report_json / write_series_json
                                  the bench CSV schema "algorithm,n,p,P,b,eps,l,r,err,t,success"
                                  and the two JSON files, byte-compatible (:26, 344-470)

What runs where: the test matrix is made (synthetic spec: fqb_gen_synthetic, the
reference's generator on the device) or loaded (load_matrix, then one upload) ONCE
and stays resident in HBM; every run reads it there.  A run's time `t` covers what
the reference's covers -- run_fixed_precision / run_fixed_rank with the SVD assembly
and the tolerance truncation -- measured on the host clock around the engine call,
which returns only once the result is ready.  `workers` > 1 runs that many engines
(one handle and CUDA stream each) from host threads, like the reference's thread
pool; each concurrent run is then timed while sharing the GPU.
"""
from __future__ import annotations

import itertools
import json
import math
import os
import threading
import time
from dataclasses import dataclass, field
from typing import List

import numpy as np

from .matrix_io import FormatError, load_matrix, matrix_format_from_name
from .rsvd import (ConfigError, Engine, FarpcaConfig, RsvdError, SketchKind, SketchSpec, ToleranceNotReached,
                   default_block, default_density, default_engine, default_max_iters, sketch_kind_from_name,
                   sketch_kind_name, truncate_to_tolerance)

CSV_HEADER = "algorithm,n,p,P,b,eps,l,r,err,t,success"
SEED_STRIDE = 0x9E3779B97F4A7C15
_U64 = (1 << 64) - 1


# ---- synthetic matrix spec (synthetic.hpp:11-22, synthetic.cpp:88-106) -------------
_SYN_KINDS = {"slow": 0, "slowdecay": 0, "fast": 1, "fastdecay": 1, "blockv": 2, "stability": 2,
              "blockvstability": 2}


def synthetic_kind_from_name(name: str) -> int:
    k = _SYN_KINDS.get(name.lower())
    if k is None:
        raise ConfigError("unknown synthetic matrix kind: " + name)
    return k


def synthetic_kind_name(kind: int) -> str:
    return {0: "slowdecay", 1: "fastdecay", 2: "blockvstability"}.get(int(kind), "unknown")


@dataclass
class SyntheticSpec:
    kind: int = 0
    n: int = 0
    d: int = 1
    seed: int = 0


# ---- config / records (experiment.hpp:16-67) --------------------------------------
@dataclass
class ExperimentConfig:
    matrix: SyntheticSpec = field(default_factory=SyntheticSpec)
    matrix_path: str = ""
    matrix_format: str = "rawf64"
    algorithms: List[SketchKind] = field(default_factory=list)
    eps: List[float] = field(default_factory=list)
    ranks: List[int] = field(default_factory=list)
    powers: List[int] = field(default_factory=lambda: [1])
    densities: List[float] = field(default_factory=lambda: [0.0])
    relative: bool = True
    block: int = 0
    max_iters: int = 0
    trials: int = 1
    seed: int = 0
    workers: int = 1
    out_prefix: str = ""


@dataclass
class RunSpec:
    kind: SketchKind = SketchKind.Gaussian
    eps: float = 0.0
    rank: int = 0
    power: int = 0
    p: float = 0.0
    seed: int = 0


@dataclass
class ExperimentRecord:
    algorithm: str = ""
    n: int = 0
    p: float = 0.0
    power: int = 0
    block: int = 0
    eps: float = 0.0
    l: int = 0          # output rank
    r: int = 0          # rank after tolerance truncation
    err: float = 0.0
    time_sec: float = 0.0
    success: bool = False
    note: str = ""      # failure detail; not part of the CSV schema


@dataclass
class ExperimentCell:
    algorithm: str = ""
    eps: float = 0.0
    rank: int = 0
    power: int = 0
    p: float = 0.0
    trials: int = 0
    mean_err: float = 0.0
    mean_time: float = 0.0
    mean_l: float = 0.0
    mean_r: float = 0.0
    success_rate: float = 0.0


@dataclass
class ExperimentReport:
    records: List[ExperimentRecord] = field(default_factory=list)
    cells: List[ExperimentCell] = field(default_factory=list)


# ---- config file --------------------------------------------------------------------
def validate_config(cfg: ExperimentConfig) -> None:
    if cfg.eps and cfg.ranks:
        raise ConfigError("config: choose an eps sweep or a rank sweep, not both")
    if not cfg.eps and not cfg.ranks:
        raise ConfigError("config: needs an eps sweep or a rank sweep")
    if any(not (e > 0.0) for e in cfg.eps):
        raise ConfigError("config: eps must be positive")
    if any(r < 1 for r in cfg.ranks):
        raise ConfigError("config: ranks must be positive")
    if any(pw < 0 for pw in cfg.powers):
        raise ConfigError("config: power must be non-negative")
    if any(p < 0.0 or p >= 1.0 for p in cfg.densities):
        raise ConfigError("config: density must lie in [0, 1)")
    if cfg.trials < 0:
        raise ConfigError("config: trials must be non-negative")
    if cfg.workers < 1:
        raise ConfigError("config: workers must be positive")
    if cfg.block < 0:
        raise ConfigError("config: block must be non-negative")
    if cfg.max_iters < 0:
        raise ConfigError("config: max_iters must be non-negative")


def _num_list(j, key, conv):
    if key not in j:
        return []
    x = j[key]
    return [conv(e) for e in x] if isinstance(x, list) else [conv(x)]


# nlohmann's get<int>() / get<double>() accept any number or boolean (static_cast);
# strings, arrays, objects and null are type errors
def _as_int(x):
    if not isinstance(x, (bool, int, float)) or (isinstance(x, float) and not math.isfinite(x)):
        raise TypeError(f"type must be number, but is {type(x).__name__}")
    return int(x)


def _as_float(x):
    if not isinstance(x, (bool, int, float)):
        raise TypeError(f"type must be number, but is {type(x).__name__}")
    return float(x)


def _as_str(x):
    if not isinstance(x, str):
        raise TypeError(f"expected a string, got {type(x).__name__}")
    return x


def _as_bool(x):
    if not isinstance(x, bool):
        raise TypeError(f"expected a boolean, got {type(x).__name__}")
    return x


def load_experiment_config(path: str | os.PathLike) -> ExperimentConfig:
    try:
        with open(path) as f:
            text = f.read()
    except OSError:
        raise ConfigError(f"cannot open config: {os.fspath(path)}") from None
    try:
        j = json.loads(text)
    except ValueError as e:
        raise ConfigError(f"config parse error: {e}") from None
    cfg = ExperimentConfig()
    try:
        if not isinstance(j, dict):
            raise TypeError(f"cannot use value() with {type(j).__name__}")
        if "matrix" in j:
            m = j["matrix"]
            if not isinstance(m, dict):
                raise TypeError(f"cannot use value() with {type(m).__name__}")
            if "path" in m:
                cfg.matrix_path = _as_str(m["path"])
                cfg.matrix_format = matrix_format_from_name(_as_str(m.get("format", "raw")))
            else:
                cfg.matrix = SyntheticSpec(synthetic_kind_from_name(_as_str(m.get("kind", "slow"))),
                                           _as_int(m.get("n", 0)), _as_int(m.get("d", 1)),
                                           _as_int(m.get("seed", 0)) & _U64)
        if "algorithms" in j:
            algs = j["algorithms"]
            cfg.algorithms = [sketch_kind_from_name(_as_str(s)) for s in (algs if isinstance(algs, list) else [algs])]
        cfg.eps = _num_list(j, "eps", _as_float)
        cfg.ranks = _num_list(j, "ranks", _as_int)
        if "power" in j:
            cfg.powers = _num_list(j, "power", _as_int)
        if "p" in j:
            cfg.densities = _num_list(j, "p", _as_float)
        cfg.relative = _as_bool(j.get("relative", True))
        cfg.block = _as_int(j.get("block", 0))
        cfg.max_iters = _as_int(j.get("max_iters", 0))
        cfg.trials = _as_int(j.get("trials", 1))
        cfg.seed = _as_int(j.get("seed", 0)) & _U64
        cfg.workers = _as_int(j.get("workers", 1))
        cfg.out_prefix = _as_str(j.get("out_prefix", ""))
    except (TypeError, AttributeError) as e:
        raise ConfigError(f"config field error: {e}") from None
    validate_config(cfg)
    return cfg


# ---- the grid (experiment.cpp:80-107) -------------------------------------------
def build_grid(cfg: ExperimentConfig) -> List[RunSpec]:
    runs: List[RunSpec] = []
    rank_mode = bool(cfg.ranks)
    epss = [0.0] if rank_mode else cfg.eps
    rks = cfg.ranks if rank_mode else [0]
    for kind in cfg.algorithms:
        for eps in epss:
            for rank in rks:
                for power in cfg.powers:
                    for p in ([0.0] if kind == SketchKind.Gaussian else cfg.densities):
                        for _ in range(cfg.trials):
                            seed = (cfg.seed + SEED_STRIDE * (len(runs) + 1)) & _U64
                            runs.append(RunSpec(SketchKind(kind), eps, rank, power, p, seed))
    return runs


# ---- one run (experiment.cpp:114-169) ----------------------------------------------
def execute_run(engine: Engine, a, m: int, n: int, norm_a: float, cfg: ExperimentConfig,
                rs: RunSpec) -> ExperimentRecord:
    rec = ExperimentRecord(algorithm=sketch_kind_name(rs.kind), n=n, power=rs.power, eps=rs.eps)
    b = cfg.block if cfg.block > 0 else default_block(m, n)
    rec.block = b
    rec.p = 0.0 if rs.kind == SketchKind.Gaussian else (rs.p if rs.p > 0.0 else default_density(rs.kind, n))
    max_iters = cfg.max_iters if cfg.max_iters > 0 else default_max_iters(n, b)
    fc = FarpcaConfig(eps=rs.eps, power=rs.power, block=b, sketch=SketchSpec(rs.kind, rec.p, rs.seed),
                      max_iters=max_iters, relative=cfg.relative)
    t0 = time.perf_counter()
    try:
        if rs.rank > 0:
            svd = engine.run_fixed_rank(a, rs.rank, fc, output="device", svd=True)
        else:
            svd = engine.run_fixed_precision(a, fc, output="device", svd=True)
    except ToleranceNotReached as e:
        svd = e.partial
        rec.note = str(e)
    except RsvdError as e:
        rec.time_sec = time.perf_counter() - t0
        rec.err = math.nan
        rec.note = str(e)
        return rec
    rec.l = svd.svd_rank()
    if rs.rank > 0:
        rec.time_sec = time.perf_counter() - t0
        rec.err = engine.relative_error(a, svd)
        rec.r = rec.l
        rec.success = not rec.note and svd.blocks < max_iters
        return rec
    eps_rel = rs.eps if cfg.relative else (rs.eps / norm_a if norm_a > 0.0 else 0.0)
    truncated = truncate_to_tolerance(svd, eps_rel, norm_a)
    rec.r = truncated.svd_rank()
    rec.time_sec = time.perf_counter() - t0
    rec.err = engine.relative_error(a, svd)
    rec.success = rec.err <= eps_rel and svd.blocks < max_iters
    return rec


# ---- aggregation (experiment.cpp:171-214) ------------------------------------------
def aggregate(records: List[ExperimentRecord], runs: List[RunSpec]) -> List[ExperimentCell]:
    cells: List[ExperimentCell] = []
    err_counts: List[int] = []
    for rec, rs in zip(records, runs):
        for idx, c in enumerate(cells):
            if (c.algorithm == rec.algorithm and c.eps == rec.eps and c.rank == rs.rank and
                    c.power == rec.power and c.p == rec.p):
                break
        else:
            cells.append(ExperimentCell(rec.algorithm, rec.eps, rs.rank, rec.power, rec.p))
            err_counts.append(0)
            idx = len(cells) - 1
        cell = cells[idx]
        cell.trials += 1
        cell.mean_time += rec.time_sec
        cell.mean_l += rec.l
        cell.mean_r += rec.r
        cell.success_rate += 1.0 if rec.success else 0.0
        if math.isfinite(rec.err):
            cell.mean_err += rec.err
            err_counts[idx] += 1
    for c, cnt in zip(cells, err_counts):
        c.mean_err = c.mean_err / cnt if cnt > 0 else 0.0
        c.mean_time /= c.trials
        c.mean_l /= c.trials
        c.mean_r /= c.trials
        c.success_rate /= c.trials
    return cells


# ---- the driver (experiment.cpp:306-315) -------------------------------------------------
def _load_input(cfg: ExperimentConfig, engine: Engine):
    """The test matrix, resident on the engine's device: (a, m, n)."""
    if cfg.matrix_path:
        import torch
        host = load_matrix(cfg.matrix_path, cfg.matrix_format)
        m, n = host.shape
        dev = torch.empty((n, m), dtype=torch.float64, device=f"cuda:{engine.device}").t()
        dev.copy_(torch.from_numpy(np.asfortranarray(host)))
        return dev, m, n
    s = cfg.matrix
    if s.n < 1:
        raise ConfigError("gen_synthetic: n must be positive")
    a, _r = engine.gen_synthetic(s.kind, s.n, s.seed, s.d)
    return a, s.n, s.n


def run_experiment(cfg: ExperimentConfig, device: int = 0, engine: Engine | None = None) -> ExperimentReport:
    validate_config(cfg)
    runs = build_grid(cfg)
    report = ExperimentReport()
    if runs:
        eng = engine if engine is not None else default_engine(device)
        a, m, n = _load_input(cfg, eng)
        norm_a = math.sqrt(eng.frob_norm_sq(a.data_ptr(), m, n, max(m, 1)))   # column-major, ld = m
        report.records = [ExperimentRecord()] * len(runs)
        extra = max(0, min(cfg.workers, len(runs)) - 1)
        engines = [eng] + [Engine(eng.device) for _ in range(extra)]
        counter, lock = itertools.count(), threading.Lock()
        failures: list = []

        def work(e: Engine):
            try:
                while True:
                    with lock:
                        i = next(counter)
                    if i >= len(runs):
                        return
                    report.records[i] = execute_run(e, a, m, n, norm_a, cfg, runs[i])
            except BaseException as exc:   # noqa: BLE001 - re-raised on the caller's thread
                failures.append(exc)

        pool = [threading.Thread(target=work, args=(e,)) for e in engines[1:]]
        for t in pool:
            t.start()
        work(engines[0])
        for t in pool:
            t.join()
        for e in engines[1:]:
            e.close()
        if failures:
            raise failures[0]
    report.cells = aggregate(report.records, runs)
    if cfg.out_prefix:
        write_report_csv(report.records, cfg.out_prefix + ".csv")
        write_report_json(report, cfg.out_prefix + ".json")
        write_series_json(report, cfg.out_prefix + "_series.json")
    return report


# ---- report files (experiment.cpp:344-470) ----------------------------------------------
def _g17(x: float) -> str:
    return "%.17g" % x


def _open_w(path):
    try:
        return open(path, "w", newline="\n")
    except OSError:
        raise FormatError(f"cannot open {os.fspath(path)} for writing", 0) from None


def write_report_csv(records: List[ExperimentRecord], path) -> None:
    with _open_w(path) as f:
        f.write(CSV_HEADER + "\n")
        for r in records:
            f.write(f"{r.algorithm},{r.n},{_g17(r.p)},{r.power},{r.block},{_g17(r.eps)},{r.l},{r.r},"
                    f"{_g17(r.err)},{_g17(r.time_sec)},{1 if r.success else 0}\n")


def _stoi(s: str) -> int:
    t = s.lstrip(" \t\n\v\f\r")
    k = 1 if t[:1] in ("+", "-") else 0
    j = k
    while j < len(t) and t[j].isdigit() and t[j].isascii():
        j += 1
    if j == k:
        raise ValueError(s)
    v = int(t[:j])
    if not -2**31 <= v < 2**31:
        raise ValueError(s)
    return v


def _stod(s: str) -> float:
    from .matrix_io import _STRTOD, _strtod_value
    t = s.lstrip(" \t\n\v\f\r").encode()
    m = _STRTOD.match(t)
    if not m:
        raise ValueError(s)
    v = _strtod_value(m.group())
    if math.isinf(v) and not m.group().lower().lstrip(b"+-").startswith(b"inf"):
        raise ValueError(s)   # std::stod throws out_of_range
    return v


def read_report_csv(path) -> List[ExperimentRecord]:
    """read_report_csv (experiment.cpp:362-416): header check, 11 columns, std::stoi /
    std::stod field parsing (leading number), FormatError with the line's byte offset."""
    try:
        with open(path, "rb") as f:
            buf = f.read().decode("latin-1")
    except OSError:
        raise FormatError(f"cannot open {os.fspath(path)}", 0) from None
    records: List[ExperimentRecord] = []
    header_seen = False
    pos = 0
    while pos < len(buf):
        eol = buf.find("\n", pos)
        if eol < 0:
            eol = len(buf)
        line, line_off = buf[pos:eol], pos
        pos = eol + 1
        if not line:
            continue
        if not header_seen:
            if line != CSV_HEADER:
                raise FormatError("unexpected report header", line_off)
            header_seen = True
            continue
        fields = line.split(",")
        if len(fields) != 11:
            raise FormatError("expected 11 report columns", line_off)
        try:
            records.append(ExperimentRecord(
                algorithm=fields[0], n=_stoi(fields[1]), p=_stod(fields[2]), power=_stoi(fields[3]),
                block=_stoi(fields[4]), eps=_stod(fields[5]), l=_stoi(fields[6]), r=_stoi(fields[7]),
                err=_stod(fields[8]), time_sec=_stod(fields[9]), success=_stoi(fields[10]) != 0))
        except ValueError:
            raise FormatError("malformed report row", line_off) from None
    if not header_seen:
        raise FormatError("empty report file", 0)
    return records


def _cell_json(c: ExperimentCell) -> dict:
    return {"algorithm": c.algorithm, "eps": c.eps, "rank": c.rank, "power": c.power, "p": c.p,
            "trials": c.trials, "mean_err": c.mean_err, "mean_time": c.mean_time, "mean_l": c.mean_l,
            "mean_r": c.mean_r, "success_rate": c.success_rate}


def _dump(obj, path) -> None:
    # the reference's JSON objects are key-sorted maps printed with a 2-space indent
    with _open_w(path) as f:
        f.write(json.dumps(obj, indent=2, sort_keys=True, ensure_ascii=False) + "\n")


def write_report_json(report: ExperimentReport, path) -> None:
    runs = []
    for r in report.records:
        d = {"algorithm": r.algorithm, "n": r.n, "p": r.p, "P": r.power, "b": r.block, "eps": r.eps, "l": r.l,
             "r": r.r, "err": r.err if math.isfinite(r.err) else None, "t": r.time_sec, "success": r.success}
        if r.note:
            d["note"] = r.note
        runs.append(d)
    _dump({"runs": runs, "cells": [_cell_json(c) for c in report.cells]}, path)


def write_series_json(report: ExperimentReport, path) -> None:
    """The swept axis is the grid dimension that actually varies (experiment.cpp:434-470)."""
    cells = report.cells

    def distinct(get):
        vals: list = []
        for c in cells:
            v = get(c)
            if v not in vals:
                vals.append(v)
        return len(vals)

    axis = "eps"
    if distinct(lambda c: float(c.rank)) > 1:
        axis = "rank"
    elif distinct(lambda c: c.p) > 1:
        axis = "p"
    elif distinct(lambda c: c.eps) > 1:
        axis = "eps"
    elif distinct(lambda c: float(c.power)) > 1:
        axis = "power"
    value_of = {"rank": lambda c: float(c.rank), "p": lambda c: c.p, "power": lambda c: float(c.power),
                "eps": lambda c: c.eps}[axis]
    series: dict = {}
    for c in cells:
        series.setdefault(c.algorithm, []).append({"x": value_of(c), "err": c.mean_err, "time": c.mean_time,
                                                   "l": c.mean_l, "success_rate": c.success_rate})
    for pts in series.values():
        pts.sort(key=lambda q: q["x"])
    _dump({"x": axis, "series": series}, path)
