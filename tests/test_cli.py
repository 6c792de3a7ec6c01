"""CLI drop-in: schema v1 validation, overrides, exit codes (CPU), and one
real run of the reference-style config on the B200 (gpu)."""

import json
import os

import pytest

from paper_2410_07381_b200 import cli

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DESK = os.path.join(ROOT, "configs", "desk_serve_train.json")


def _write(tmp_path, doc, name="cfg.json"):
    p = tmp_path / name
    p.write_text(json.dumps(doc))
    return str(p)


def test_bad_schema_and_json_exit_2(tmp_path):
    assert cli.main(["run", "--config", _write(tmp_path, {"schema_version": 2}), "--out",
                     str(tmp_path / "o")]) == cli.EXIT_CONFIG
    bad = tmp_path / "bad.json"
    bad.write_text("{not json")
    assert cli.main(["run", "--config", str(bad), "--out", str(tmp_path / "o")]) == cli.EXIT_CONFIG
    assert cli.main(["run", "--config", str(tmp_path / "missing.json"), "--out", "x"]) == cli.EXIT_CONFIG
    assert cli.main(["frobnicate"]) == cli.EXIT_CONFIG


def test_validation_errors(tmp_path):
    doc = json.load(open(DESK))
    for patch in ({"policies": ["Fifo"]}, {"duration_s": 0},
                  {"gpu": {"num_sms": 0, "max_threads_per_sm": 1, "max_blocks_per_sm": 1}}):
        d = {**doc, **patch}
        with pytest.raises(cli.ConfigError):
            cli.validate(d)
    d = json.loads(json.dumps(doc))
    d["workloads"][0]["priority"] = "urgent"
    with pytest.raises(cli.ConfigError):
        cli.validate(d)
    d = json.loads(json.dumps(doc))
    del d["workloads"][1]["kernels"][0]["total_blocks"]
    with pytest.raises(cli.ConfigError):
        cli.validate(d)
    cli.validate(doc)


def test_overrides_and_hash(tmp_path):
    import argparse
    doc = json.load(open(DESK))
    o = cli.apply_overrides(doc, argparse.Namespace(policy="Eager", threshold_ms=0.1, seed=7,
                                                    duration_s=2.0, load=0.3, trace=None))
    assert o["policies"] == ["Eager"] and o["scheduler"]["threshold_ms"] == 0.1
    assert o["seed"] == 7 and o["duration_s"] == 2.0
    assert o["workloads"][0]["trace"] == {"load": 0.3, "seed": 0}
    o2 = cli.apply_overrides(doc, argparse.Namespace(trace="t.csv"))
    assert o2["workloads"][0]["trace"] == {"seed": 0, "path": "t.csv"}
    assert cli.config_sha256(doc) == cli.config_sha256(json.loads(json.dumps(doc)))
    assert cli.config_sha256(doc) != cli.config_sha256(o)
    assert doc["policies"] == ["Tally", "KernelPriority", "Eager"]      # input untouched


@pytest.mark.gpu
def test_run_desk_config_on_b200(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    out = tmp_path / "out"
    rc = cli.main(["run", "--config", DESK, "--out", str(out), "--duration-s", "0.3", "--events"])
    assert rc == cli.EXIT_OK
    rows = (out / "metrics.csv").read_text().strip().splitlines()
    assert rows[0] == "policy,task,p99_ms,norm_throughput,system_throughput"
    assert {r.split(",")[0] for r in rows[1:]} == {"Tally", "KernelPriority", "Eager"}
    man = json.loads((out / "manifest.json").read_text())
    doc = cli.apply_overrides(json.load(open(DESK)), type("A", (), {"duration_s": 0.3})())
    assert man["config_sha256"] == cli.config_sha256(doc)
    assert (out / "events_Tally.csv").read_text().startswith("time_ns,kind,task,kernel,block")
