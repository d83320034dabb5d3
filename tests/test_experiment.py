"""Experiment driver host logic (paper_2506_03859_b200/experiment.py) pinned against the
reference's own experiment.cpp, run here on the CPU through oracle/_ref:

* the config loader's validation (same ConfigError messages),
* the report CSV writer / reader (byte-identical files, same FormatError offsets),
* aggregate + write_report_json + write_series_json: fed the reference's own
  records, our files must equal the reference's byte for byte.
"""
import json
import math

import pytest

from paper_2506_03859_b200 import ConfigError, FormatError
from paper_2506_03859_b200 import experiment as ex

GRID_FP = {"matrix": {"kind": "slow", "n": 160, "seed": 11}, "algorithms": ["gaussian", "sparsesign", "stdbernoulli"],
           "eps": [1e-2, 3e-3], "power": [1], "p": [0.0, 0.05], "block": 10, "trials": 2, "seed": 5}
GRID_RANK = {"matrix": {"kind": "fast", "n": 120, "seed": 3}, "algorithms": ["gaussian", "bernoulli"],
             "ranks": [10, 25], "power": [0, 2], "block": 10, "seed": 1, "relative": False}
GRID_UNREACHABLE = {"matrix": {"kind": "slow", "n": 100, "seed": 2}, "algorithms": ["sparsegaussian"],
                    "eps": [1e-9], "power": 1, "block": 10, "max_iters": 2}


def _write_cfg(tmp_path, cfg, name="cfg.json"):
    p = tmp_path / name
    p.write_text(json.dumps(cfg))
    return p


def _run_reference(reference, tmp_path, cfg, tag):
    prefix = str(tmp_path / f"ref_{tag}")
    path = _write_cfg(tmp_path, dict(cfg, out_prefix=prefix), f"{tag}.json")
    assert reference.run_experiment(path) is None
    return prefix, path


@pytest.mark.parametrize("tag,cfg", [("fp", GRID_FP), ("rank", GRID_RANK), ("tol", GRID_UNREACHABLE)])
def test_report_files_match_reference(reference, tmp_path, tag, cfg):
    prefix, cfg_path = _run_reference(reference, tmp_path, cfg, tag)
    records = ex.read_report_csv(prefix + ".csv")
    n, err = reference.read_report_csv(prefix + ".csv")
    assert err is None and n == len(records)
    # notes are JSON-only; take them from the reference's runs
    ref_json = json.loads(open(prefix + ".json").read())
    for rec, run in zip(records, ref_json["runs"]):
        rec.note = run.get("note", "")
    mine = ex.load_experiment_config(cfg_path)
    runs = ex.build_grid(mine)
    assert len(runs) == len(records)
    report = ex.ExperimentReport(records, ex.aggregate(records, runs))
    out = str(tmp_path / f"ours_{tag}")
    ex.write_report_csv(report.records, out + ".csv")
    ex.write_report_json(report, out + ".json")
    ex.write_series_json(report, out + "_series.json")
    for suffix in (".csv", ".json", "_series.json"):
        assert open(out + suffix, "rb").read() == open(prefix + suffix, "rb").read(), suffix


def test_grid_order_and_seeds():
    cfg = ex.ExperimentConfig(algorithms=[0, 3], eps=[1e-2, 1e-3], powers=[1, 2], densities=[0.0, 0.1], trials=2,
                              seed=2**64 - 3)
    runs = ex.build_grid(cfg)
    # gaussian ignores the density sweep: 2 eps x 2 powers x 1 x 2 trials; sparse sign: x2 densities
    assert len(runs) == 8 + 16
    assert [r.kind for r in runs[:8]] == [0] * 8 and runs[8].kind == 3
    assert (runs[0].eps, runs[0].power, runs[0].p) == (1e-2, 1, 0.0)
    assert (runs[2].eps, runs[2].power) == (1e-2, 2)
    assert all(r.seed == (cfg.seed + ex.SEED_STRIDE * (i + 1)) % 2**64 for i, r in enumerate(runs))
    assert runs[8].p == 0.0 and runs[10].p == 0.1


BAD_CONFIGS = [
    ({"algorithms": ["gaussian"]}, "config: needs an eps sweep or a rank sweep"),
    ({"eps": 0.1, "ranks": [3]}, "config: choose an eps sweep or a rank sweep, not both"),
    ({"eps": [0.1, 0.0]}, "config: eps must be positive"),
    ({"ranks": [0]}, "config: ranks must be positive"),
    ({"eps": 0.1, "power": -1}, "config: power must be non-negative"),
    ({"eps": 0.1, "p": [0.5, 1.0]}, "config: density must lie in [0, 1)"),
    ({"eps": 0.1, "trials": -1}, "config: trials must be non-negative"),
    ({"eps": 0.1, "workers": 0}, "config: workers must be positive"),
    ({"eps": 0.1, "block": -2}, "config: block must be non-negative"),
    ({"eps": 0.1, "max_iters": -1}, "config: max_iters must be non-negative"),
    ({"eps": 0.1, "algorithms": ["gauss"]}, "unknown sketch kind: gauss"),
    ({"eps": 0.1, "matrix": {"kind": "medium"}}, "unknown synthetic matrix kind: medium"),
    ({"eps": 0.1, "matrix": {"path": "x", "format": "csv"}}, "unknown matrix format: csv"),
    ({"eps": "tight"}, "config field error: "),
    ({"eps": 0.1, "relative": 1}, "config field error: "),
]


@pytest.mark.parametrize("cfg,msg", BAD_CONFIGS)
def test_config_validation_matches_reference(reference, tmp_path, cfg, msg):
    path = _write_cfg(tmp_path, cfg)
    st = reference.check_experiment_config(path)
    assert st is not None and st[0] == 2 and st[1].startswith(msg)
    with pytest.raises(ConfigError) as e:
        ex.load_experiment_config(path)
    assert str(e.value).startswith(msg)
    if not msg.endswith(": "):
        assert str(e.value) == st[1]


def test_config_parse_errors(tmp_path):
    p = tmp_path / "bad.json"
    p.write_text("{not json")
    with pytest.raises(ConfigError, match="config parse error"):
        ex.load_experiment_config(p)
    with pytest.raises(ConfigError, match="cannot open config"):
        ex.load_experiment_config(tmp_path / "missing.json")


def test_config_defaults_and_scalars(tmp_path):
    cfg = ex.load_experiment_config(_write_cfg(tmp_path, {"eps": 0.05, "power": 2, "p": 0.1, "seed": -1}))
    assert cfg.eps == [0.05] and cfg.powers == [2] and cfg.densities == [0.1]
    assert cfg.seed == 2**64 - 1 and cfg.relative and cfg.trials == 1 and cfg.workers == 1
    assert cfg.matrix.kind == 0 and cfg.matrix.d == 1 and cfg.matrix_path == ""


CSV_HEADER = "algorithm,n,p,P,b,eps,l,r,err,t,success\n"
BAD_CSV = [
    ("", "empty report file"),
    ("algorithm,n\n", "unexpected report header"),
    (CSV_HEADER + "gaussian,1,0,1,10,0.1,10,10,0.5,0.1\n", "expected 11 report columns"),
    (CSV_HEADER + "gaussian,x,0,1,10,0.1,10,10,0.5,0.1,1\n", "malformed report row"),
    (CSV_HEADER + "gaussian,1,0,1,10,0.1,10,10,1e999,0.1,1\n", "malformed report row"),
]


@pytest.mark.parametrize("text,msg", BAD_CSV)
def test_csv_reader_errors_match_reference(reference, tmp_path, text, msg):
    p = tmp_path / "r.csv"
    p.write_text(text)
    _, ref_err = reference.read_report_csv(p)
    with pytest.raises(FormatError) as e:
        ex.read_report_csv(p)
    assert ref_err == (1, e.value.msg, e.value.offset) and e.value.msg == msg


def test_csv_reader_lenient_fields_match_reference(reference, tmp_path):
    """std::stoi / std::stod read a leading number and ignore the rest, like the reference."""
    p = tmp_path / "r.csv"
    p.write_text(CSV_HEADER + "\ngaussian, 7x,0.5e0junk,1,10,1e-2,10,9,nan,inf,2\n")
    n, err = reference.read_report_csv(p)
    recs = ex.read_report_csv(p)
    assert err is None and n == len(recs) == 1
    r = recs[0]
    assert (r.n, r.p, r.l, r.r, r.success) == (7, 0.5, 10, 9, True)
    assert math.isnan(r.err) and math.isinf(r.time_sec)
