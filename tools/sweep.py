#!/usr/bin/env python
"""Kernel-variant sweeps without touching the product library.

  # here (CPU): build variants of libasse with compile-time knobs into tools/variants/
  python tools/sweep.py build nb4 -D ASSE_OWN_NB=4
  python tools/sweep.py build def
  # on the GPU box: bench every variant on every workload, interleaved, R repetitions
  python tools/sweep.py run --variants def,nb4 --workloads C5,C3 --reps 2

Each run loads its variant through ASSE_LIB (paper_1807_01527_b200/asse.py); the product
paper_1807_01527_b200/libasse.so is never overwritten. Results: one JSON line per run in
gpurun_out/sweep_<tag>.jsonl and a table on stdout."""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
VAR = os.path.join(ROOT, "tools", "variants")


def cmd_build(a):
    sys.path.insert(0, ROOT)
    from paper_1807_01527_b200 import _build
    os.makedirs(VAR, exist_ok=True)
    out = os.path.join(VAR, "libasse_%s.so" % a.name)
    _build.build_variant(out, a.D or [], verbose=a.verbose)
    print(out)


def cmd_run(a):
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    log = os.path.join(ROOT, "gpurun_out", "sweep_%s.jsonl" % a.tag)
    rows = []
    with open(log, "a") as f:
        for rep in range(a.reps):
            for w in a.workloads.split(","):
                for v in a.variants.split(","):
                    lib = os.path.join(VAR, "libasse_%s.so" % v)
                    env = dict(os.environ, ASSE_LIB=lib)
                    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--workload", w, "--steps", str(a.steps),
                           "--warmup", "3", "--no-e2e", "--no-cpu", "--scan-variant", str(a.scan_variant)]
                    try:
                        out = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=a.timeout)
                        line = [x for x in out.stdout.splitlines() if x.startswith("{")][-1]
                        d = json.loads(line)
                        row = dict(variant=v, workload=w, rep=rep, gpps=d["value"], ms_per_step=d["ms_per_step"],
                                   scan_ms=d["roofline"]["avg_launch_ms"], end_slice_ms=d["end_slice_ms"],
                                   fold_ms=d["kernels"]["k_fold"]["avg_launch_ms"], clocks=d["clocks"])
                    except Exception as e:  # keep sweeping
                        row = dict(variant=v, workload=w, rep=rep, error=repr(e)[:300])
                    rows.append(row)
                    f.write(json.dumps(row) + "\n")
                    f.flush()
                    print(json.dumps({k: row[k] for k in row if k != "clocks"}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    sub = ap.add_subparsers(dest="cmd", required=True)
    b = sub.add_parser("build")
    b.add_argument("name")
    b.add_argument("-D", action="append")
    b.add_argument("-v", "--verbose", action="store_true")
    r = sub.add_parser("run")
    r.add_argument("--variants", required=True)
    r.add_argument("--workloads", default="C5")
    r.add_argument("--reps", type=int, default=1)
    r.add_argument("--steps", type=int, default=20)
    r.add_argument("--scan-variant", type=int, default=0)
    r.add_argument("--timeout", type=int, default=600)
    r.add_argument("--tag", default="run")
    a = ap.parse_args()
    cmd_build(a) if a.cmd == "build" else cmd_run(a)


if __name__ == "__main__":
    main()
