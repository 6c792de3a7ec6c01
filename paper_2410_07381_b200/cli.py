"""Command line, drop-in for the reference's ``tallysim`` CLI on the B200.

    python -m paper_2410_07381_b200 run     --config cfg.json --out DIR [overrides]
    python -m paper_2410_07381_b200 profile --config cfg.json --out DIR
    python -m paper_2410_07381_b200 sweep   --config cfg.json --out DIR --axis threshold|load|be-count
    python -m paper_2410_07381_b200 interpret --kernel k.json --memory mem.json --args 0 8 16 [--shape ptb --workers 4]

Config: the reference's JSON schema v1 (ref cli.py:58, :95-247): ``gpu``,
``workloads`` (kernels as cost models), ``policies``, ``scheduler``
(threshold_ms, quantum_ms), ``seed``, ``duration_s``.  On the B200 every
``KernelWork`` runs as a ``spin`` cost-model kernel with the model's blocks,
threads and block duration in all three shapes, scheduled in real time by the
native runner; ``gpu`` in the config is informational (the device's real
GpuSpec is used).  Outputs mirror the reference: ``metrics.csv``
(``policy,task,p99_ms,norm_throughput,system_throughput``), ``profile_cache.json``,
optional ``events.csv``, and ``manifest.json`` with the config's sha256
(ref cli.py:250-264).  Exit codes: 0 ok, 1 runtime error, 2 invalid
config/arguments, 3 transformation refused (ref cli.py:53-56).
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import tempfile

EXIT_OK, EXIT_RUNTIME, EXIT_CONFIG, EXIT_TRANSFORM = 0, 1, 2, 3
SCHEMA_VERSION = 1
THRESHOLD_GRID_MS = (0.01, 0.0316, 0.1, 0.316, 1.0, 3.16, 10.0)   # ref cli.py:60


class ConfigError(ValueError):
    pass


def _need(doc, key, where):
    if key not in doc:
        raise ConfigError(f"{where}: missing required key {key!r}")
    return doc[key]


def load_config(path):
    try:
        doc = json.load(open(path))
    except OSError as e:
        raise ConfigError(f"cannot read config {path}: {e}") from None
    except json.JSONDecodeError as e:
        raise ConfigError(f"{path}: invalid JSON: {e}") from None
    if not isinstance(doc, dict) or doc.get("schema_version") != SCHEMA_VERSION:
        raise ConfigError(f"{path}: expected a JSON object with schema_version {SCHEMA_VERSION}")
    return doc


def config_sha256(doc) -> str:
    return hashlib.sha256(json.dumps(doc, sort_keys=True, separators=(",", ":")).encode()).hexdigest()


def apply_overrides(doc, args):
    doc = json.loads(json.dumps(doc))
    if getattr(args, "policy", None):
        doc["policies"] = [args.policy]
    if getattr(args, "threshold_ms", None) is not None:
        doc.setdefault("scheduler", {})["threshold_ms"] = args.threshold_ms
    if getattr(args, "seed", None) is not None:
        doc["seed"] = args.seed
    if getattr(args, "duration_s", None) is not None:
        doc["duration_s"] = args.duration_s
    for key, val in (("load", getattr(args, "load", None)), ("path", getattr(args, "trace", None))):
        if val is None:
            continue
        hit = False
        for wl in doc.get("workloads", []):
            if wl.get("kind") == "inference":
                tr = wl.setdefault("trace", {})
                tr.pop("load" if key == "path" else "path", None)
                tr[key] = val
                hit = True
        if not hit:
            raise ConfigError("no inference workload to apply the trace override to")
    return doc


def build_workloads(doc, spin_kernels=True):
    """Schema v1 workloads -> WorkloadSpecs whose KernelWorks carry ``spin``
    device kernels (one per kernel_id)."""
    from . import device as D
    from . import kernels as K
    from .scheduler import KernelWork
    from .workloads import TraceSpec, WorkloadSpec
    dev_kernels = {}
    out = []
    for w in _need(doc, "workloads", "config"):
        name = str(_need(w, "name", "workload"))
        where = f"workload {name!r}"
        prio = {"high": D.HIGH, "best_effort": D.BEST_EFFORT}.get(str(_need(w, "priority", where)).lower())
        if prio is None:
            raise ConfigError(f"{where}: priority must be high or best_effort")
        works = []
        for i, kd in enumerate(_need(w, "kernels", where)):
            kw = f"{where} kernel {i}"
            try:
                cost = D.cost_model(float(_need(kd, "block_duration_ms", kw)), int(_need(kd, "total_blocks", kw)),
                                    int(kd.get("threads_per_block", 32)), kd.get("launch_overhead_ms"),
                                    kd.get("ptb_iteration_overhead_ms"))
            except ValueError as e:
                raise ConfigError(f"{kw}: {e}") from None
            kid = str(_need(kd, "kernel_id", kw))
            dk = None
            if spin_kernels:
                if kid not in dev_kernels:
                    dev_kernels[kid] = K.spin(cost.total_blocks, cost.threads_per_block,
                                              cost.block_duration_ns)
                dk = dev_kernels[kid]
            works.append(KernelWork(kid, cost, bool(kd.get("exempt", False)), kernel=dk))
        trace = None
        if w.get("trace") is not None:
            t = w["trace"]
            try:
                trace = TraceSpec(load=t.get("load"), seed=int(t.get("seed", 0)), path=t.get("path"),
                                  rescale=float(t.get("rescale", 1.0)))
            except ValueError as e:
                raise ConfigError(f"{where}: trace: {e}") from None
        try:
            out.append(WorkloadSpec(name, str(_need(w, "kind", where)), prio, tuple(works), trace))
        except ValueError as e:
            raise ConfigError(f"{where}: {e}") from None
    return out


def validate(doc):
    """Everything checkable without a device (exit code 2 on failure)."""
    from .scheduler import POLICIES
    build_workloads(doc, spin_kernels=False)
    for p in doc.get("policies", ["Tally"]):
        if p not in POLICIES:
            raise ConfigError(f"unknown policy {p!r} (choose from {', '.join(POLICIES)})")
    if float(doc.get("duration_s", 10.0)) <= 0:
        raise ConfigError("duration_s must be > 0")
    g = doc.get("gpu")
    if g is not None:
        from .device import GpuSpec
        try:
            GpuSpec(int(_need(g, "num_sms", "gpu")), int(_need(g, "max_threads_per_sm", "gpu")),
                    int(_need(g, "max_blocks_per_sm", "gpu")))
        except ValueError as e:
            raise ConfigError(f"gpu: {e}") from None


def _atomic_write(path, text):
    d = os.path.dirname(os.path.abspath(path))
    fd, tmp = tempfile.mkstemp(dir=d, prefix=".tmp-")
    with os.fdopen(fd, "w") as fh:
        fh.write(text)
    os.replace(tmp, path)


def _manifest(out_dir, command, doc, outputs):
    m = {"command": command, "config_sha256": config_sha256(doc), "seed": doc.get("seed", 0),
         "outputs": sorted(outputs), "device": "B200"}
    _atomic_write(os.path.join(out_dir, "manifest.json"), json.dumps(m, indent=2, sort_keys=True) + "\n")


def _experiment(doc, record_events=False, profiler=None):
    from .device import B200Device, ms_to_ns
    from .profiler import Profiler
    from .scheduler import POLICIES
    from .workloads import run_experiment
    validate(doc)
    dev = B200Device.get(0)
    wls = build_workloads(doc)
    pols = list(doc.get("policies", ["Tally"]))
    dur = float(doc.get("duration_s", 10.0))
    sch = doc.get("scheduler", {})
    th, q = sch.get("threshold_ms"), sch.get("quantum_ms")
    prof = profiler or Profiler(dev.spec, runs=int(doc.get("profile_runs", 5)))
    for wl in wls:
        for w in wl.kernels:
            prof.bind(w.kernel_id, w.kernel)
    reps = run_experiment(dev.spec, wls, pols, ms_to_ns(dur * 1000.0), seed=int(doc.get("seed", 0)),
                          turnaround_threshold_ns=None if th is None else ms_to_ns(float(th)),
                          quantum_ns=None if q is None else ms_to_ns(float(q)),
                          record_events=record_events, profiler=prof)
    return reps, prof


def cmd_run(args):
    from .device import events_to_csv
    from .workloads import CSV_HEADER, report_csv_rows
    doc = apply_overrides(load_config(args.config), args)
    os.makedirs(args.out, exist_ok=True)
    reps, prof = _experiment(doc, record_events=args.events)
    rows = [CSV_HEADER] + [r for rep in reps for r in report_csv_rows(rep)]
    outs = ["metrics.csv", "profile_cache.json"]
    _atomic_write(os.path.join(args.out, "metrics.csv"), "\n".join(rows) + "\n")
    _atomic_write(os.path.join(args.out, "profile_cache.json"), prof.dump_cache())
    if args.events:
        for rep in reps:
            name = f"events_{rep.policy}.csv"
            _atomic_write(os.path.join(args.out, name), events_to_csv(rep.result.events))
            outs.append(name)
    _manifest(args.out, "run", doc, outs)
    print("\n".join(rows))
    return EXIT_OK


def cmd_profile(args):
    from .device import B200Device
    from .profiler import Profiler
    doc = load_config(args.config)
    os.makedirs(args.out, exist_ok=True)
    dev = B200Device.get(0)
    prof = Profiler(dev.spec, runs=int(doc.get("profile_runs", 5)))
    for wl in build_workloads(doc):
        for w in wl.kernels:
            prof.bind(w.kernel_id, w.kernel)
            prof.profile(w.profile_key(), w.cost)
    _atomic_write(os.path.join(args.out, "profile_cache.json"), prof.dump_cache())
    _manifest(args.out, "profile", doc, ["profile_cache.json"])
    return EXIT_OK


def cmd_sweep(args):
    from .workloads import CSV_HEADER, report_csv_rows
    base = load_config(args.config)
    os.makedirs(args.out, exist_ok=True)
    rows = ["axis_value," + CSV_HEADER]
    if args.axis == "threshold":
        points = [(v, {"scheduler": {**base.get("scheduler", {}), "threshold_ms": v}}) for v in THRESHOLD_GRID_MS]
    elif args.axis == "load":
        points = []
        for v in (0.1, 0.3, 0.5, 0.7, 0.9):
            d = apply_overrides(base, argparse.Namespace(load=v))
            points.append((v, {"workloads": d["workloads"]}))
    else:
        be = [w for w in base["workloads"] if str(w.get("priority", "")).lower() == "best_effort"]
        if not be:
            raise ConfigError("be-count sweep needs a best_effort workload")
        points = []
        for n in range(1, int(args.max_be) + 1):
            others = [w for w in base["workloads"] if w not in be]
            copies = [dict(be[0], name=f"{be[0]['name']}{i}") for i in range(n)]
            points.append((n, {"workloads": others + copies}))
    for v, patch in points:
        doc = {**base, **patch}
        reps, _ = _experiment(doc)
        rows += [f"{v}," + r for rep in reps for r in report_csv_rows(rep)]
    _atomic_write(os.path.join(args.out, "sweep.csv"), "\n".join(rows) + "\n")
    _manifest(args.out, f"sweep {args.axis}", base, ["sweep.csv"])
    print("\n".join(rows))
    return EXIT_OK


def cmd_interpret(args):
    """Run an IR kernel (JSON encoding) on the B200 via IR-JIT."""
    import torch
    from . import irjit
    k = json.load(open(args.kernel))
    mem = json.load(open(args.memory))
    jk = irjit.JitKernel(k)
    m = torch.tensor(mem, dtype=torch.int64, device="cuda")
    fault = torch.zeros(1, dtype=torch.int64, device="cuda")
    dk = jk.bind(m, fault, tuple(int(a) for a in args.args))
    from .kernels import Stream
    s = Stream(high_priority=False)
    if args.shape == "ptb":
        dk.ptb(s, args.workers).wait()
    elif args.shape == "sliced":
        from .transforms import slice_plan
        from fractions import Fraction
        for o, g in slice_plan(None, Fraction(args.fraction), grid=k["grid"]):
            dk.sliced_rect(s, o, g).wait()
    else:
        dk.original(s).wait()
    torch.cuda.synchronize()
    status = "Completed" if int(fault.item()) == 0 else ("StepLimitExceeded" if int(fault.item()) & 2 else "MemoryFault")
    print(json.dumps({"status": status, "memory": m.cpu().tolist() if status == "Completed" else None}))
    return EXIT_OK if status == "Completed" else EXIT_RUNTIME


def main(argv=None):
    ap = argparse.ArgumentParser(prog="paper_2410_07381_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    r = sub.add_parser("run")
    r.add_argument("--config", required=True)
    r.add_argument("--out", required=True)
    r.add_argument("--policy")
    r.add_argument("--threshold-ms", type=float)
    r.add_argument("--seed", type=int)
    r.add_argument("--duration-s", type=float)
    r.add_argument("--load", type=float)
    r.add_argument("--trace")
    r.add_argument("--events", action="store_true")
    p = sub.add_parser("profile")
    p.add_argument("--config", required=True)
    p.add_argument("--out", required=True)
    s = sub.add_parser("sweep")
    s.add_argument("--config", required=True)
    s.add_argument("--out", required=True)
    s.add_argument("--axis", choices=["threshold", "load", "be-count"], required=True)
    s.add_argument("--max-be", type=int, default=4)
    i = sub.add_parser("interpret")
    i.add_argument("--kernel", required=True)
    i.add_argument("--memory", required=True)
    i.add_argument("--args", nargs="*", default=[])
    i.add_argument("--shape", choices=["original", "sliced", "ptb"], default="original")
    i.add_argument("--workers", type=int, default=4)
    i.add_argument("--fraction", default="1/4")
    try:
        args = ap.parse_args(argv)
    except SystemExit as e:
        return EXIT_CONFIG if e.code else EXIT_OK
    try:
        return {"run": cmd_run, "profile": cmd_profile, "sweep": cmd_sweep,
                "interpret": cmd_interpret}[args.cmd](args)
    except ConfigError as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_CONFIG
    except ValueError as e:
        from .transforms import TransformError
        print(f"error: {e}", file=sys.stderr)
        return EXIT_TRANSFORM if isinstance(e, TransformError) else EXIT_CONFIG
    except Exception as e:   # runtime failure (device, CUDA)
        print(f"error: {e}", file=sys.stderr)
        return EXIT_RUNTIME
