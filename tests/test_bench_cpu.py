"""bench.py on the CPU: the reference arm runs the same configuration as the
B200 arm (identical ``config`` object, same arrival traces) and pools its p99
over every window; the multi-pair launcher aggregates per-pair results."""

import json
import os
import subprocess
import sys
from types import SimpleNamespace

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def _args(**kw):
    a = dict(config="c2", steps=2, warmup=0, gpus=1, load=0.5, burst=20.0, burst_gaps=2.0, window_ms=300.0,
             threshold_us=31.6, batch=64, gen=16, ref_profile_runs=1, lookahead=4)
    a.update(kw)
    return SimpleNamespace(**a)


def test_run_config_is_a_function_of_the_arguments():
    a, b = _args(), _args()
    assert bench.run_config(a) == bench.run_config(b)
    assert bench.run_config(_args(steps=3))["trace_seeds"] == [0, 1, 2]
    assert bench.run_config(_args(load=0.25)) != bench.run_config(a)


def test_reference_arm_same_config_and_pooled_p99():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "c2",
                          "--window-ms", "300", "--steps", "3", "--warmup", "1", "--ref-profile-runs", "1"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    args = _args(steps=3, warmup=1, window_ms=300.0)
    assert line["config"] == json.loads(json.dumps(bench.run_config(args)))
    assert line["e2e"]["h2d_bytes_per_step"] == 0
    cb = line["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["sim_ms_per_wall_s"] > 0
    assert line["components"]["requests"] > 0
    assert line["value"] is not None


def test_reference_traces_are_the_gpu_arms():
    """Both arms draw window k's arrivals from c2_trace(seed=k) at the
    committed isolated latency: the traces are the same objects."""
    costs = json.load(open(bench.costs_path("c2")))
    lat = int(costs["hp_latency_ns"])
    a = bench.c2_trace(0.5, lat, int(300e6), 0, 20.0, 2.0)
    b = bench.c2_trace(0.5, lat, int(300e6), 0, 20.0, 2.0)
    assert a == b and len(a) > 0 and all(x < 300e6 for x in a)


def test_gpus_n_spawns_independent_pairs():
    """`bench.py --gpus 2` without torchrun: two pair processes joined by a
    gloo control-plane group (no NCCL); rank 0 reports both pairs."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--selftest-pairs"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT,
                         env={k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK")})
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2
    per = line["components"]["per_rank"]
    assert [d["rank"] for d in per] == [0, 1]
    assert line["value"] == 1.0                      # the worst pair
    assert line["components"]["be_throughput_pct"] == 99.0
    assert line["ms_per_step"] >= 11.0               # max over ranks (rank 1 sleeps 11 ms)


def test_gpus_n_under_torchrun_uses_gloo():
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", str(bench.free_port()),
                          os.path.join(ROOT, "bench.py"), "--gpus", "2", "--selftest-pairs"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == 2 and len(line["components"]["per_rank"]) == 2
