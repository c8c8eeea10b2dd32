"""Command line of the reference (tools/main.cpp) over the GPU pipeline:

  python -m paper_2601_04422_b200 run --qasm FILE [--sidecar F] [--backend mps-serial|mps-parallel|statevector]
        [--nonlocal swap|bondprop] [--max-bond N] [--cutoff X] [--shots N] [--seed N] [--workers N]
        [--deterministic] [--no-memoize] [--cache-cap N] [--out FILE] [--device N]
  python -m paper_2601_04422_b200 gen-ghz --n N [--measure] [--out FILE]
  python -m paper_2601_04422_b200 gen-brickwork --n N --depth D [--seed S] [--measure] [--entangler cx|haar]
        [--out FILE]
  python -m paper_2601_04422_b200 bench [--circuit ghz|brickwork] --sweep-n N... [--sweep-max-bond B...]
        [--backends B...] [--depth D] [--seed S] [--repeat R] [--out FILE]

Errors print "error: <message>" and exit with exit_code_for_error's code
(config 1, parse 2, numeric 3; runner.cpp:330-341).
"""
from __future__ import annotations

import argparse
import json
import os
import sys

from . import frontend as F


def _emit(obj, path):
    text = json.dumps(obj, indent=2) + "\n"
    if path:
        with open(path, "w") as f:
            f.write(text)
    else:
        sys.stdout.write(text)


def _write(text, path):
    if path:
        with open(path, "w") as f:
            f.write(text)
    else:
        sys.stdout.write(text)


def _workers(flag, deterministic):  # resolve_workers, tools/main.cpp:60-80
    if deterministic:
        return 1
    if flag is not None:
        return flag
    env = os.environ.get("MPSIM_WORKERS")
    return int(env) if env else max(1, os.cpu_count() or 1)


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="mpsim", description="Matrix-product-state quantum circuit simulator (B200)")
    sub = ap.add_subparsers(dest="cmd", required=True)
    r = sub.add_parser("run", help="Simulate a QASM file")
    r.add_argument("--qasm", required=True)
    r.add_argument("--sidecar", default="")
    r.add_argument("--backend", default="mps-serial")
    r.add_argument("--nonlocal", dest="nonlocal_", default="swap")
    r.add_argument("--max-bond", type=int, default=0)
    r.add_argument("--cutoff", type=float, default=0.0)
    r.add_argument("--shots", type=int, default=0)
    r.add_argument("--seed", type=int, default=1)
    r.add_argument("--workers", type=int, default=None)
    r.add_argument("--deterministic", action="store_true")
    r.add_argument("--no-memoize", action="store_true")
    r.add_argument("--cache-cap", type=int, default=0)
    r.add_argument("--out", default="")
    r.add_argument("--device", type=int, default=0)
    g = sub.add_parser("gen-ghz", help="Generate a GHZ circuit")
    g.add_argument("--n", type=int, required=True)
    g.add_argument("--measure", action="store_true")
    g.add_argument("--out", default="")
    b = sub.add_parser("gen-brickwork", help="Generate a brickwork circuit")
    b.add_argument("--n", type=int, required=True)
    b.add_argument("--depth", type=int, required=True)
    b.add_argument("--seed", type=int, default=1)
    b.add_argument("--measure", action="store_true")
    b.add_argument("--entangler", default="cx")
    b.add_argument("--out", default="")
    s = sub.add_parser("bench", help="Sweep benchmark runs")
    s.add_argument("--circuit", default="ghz")
    s.add_argument("--sweep-n", type=int, nargs="+", required=True)
    s.add_argument("--sweep-max-bond", type=int, nargs="+", default=[0])
    s.add_argument("--backends", nargs="+", default=["mps-serial"])
    s.add_argument("--depth", type=int, default=10)
    s.add_argument("--seed", type=int, default=1)
    s.add_argument("--repeat", type=int, default=1)
    s.add_argument("--out", default="")
    a = ap.parse_args(argv)
    try:
        if a.cmd == "run":
            rec = F.run_circuit(qasm_path=a.qasm, sidecar_path=a.sidecar or None, backend=a.backend,
                                nonlocal_method=a.nonlocal_, max_bond=a.max_bond, cutoff=a.cutoff, shots=a.shots,
                                seed=a.seed,
                                workers=_workers(a.workers, a.deterministic) if a.backend == "mps-parallel" else 1,
                                memoize=not a.no_memoize, cache_cap=a.cache_cap, device=a.device)
            _emit(rec, a.out)
        elif a.cmd == "gen-ghz":
            _write(F.ghz_qasm(a.n, a.measure), a.out)
        elif a.cmd == "gen-brickwork":
            if a.entangler == "haar" and not a.out:
                raise F.ConfigError("--entangler haar needs --out to place the sidecar file")
            qasm, sc = F.brickwork_qasm(a.n, a.depth, a.seed, a.measure, a.entangler)
            _write(qasm, a.out)
            if sc:
                with open(a.out + ".u4.json", "w") as f:
                    f.write(json.dumps(json.loads(sc), indent=2) + "\n")
                print(a.out + ".u4.json")
        else:
            if a.circuit not in ("ghz", "brickwork"):
                raise F.ConfigError(f"unknown bench circuit '{a.circuit}'")
            recs = []
            for n in a.sweep_n:
                if a.circuit == "ghz":
                    text, label = F.ghz_qasm(n), f"ghz-{n}"
                else:
                    text, label = F.brickwork_qasm(n, a.depth, a.seed)[0], f"brickwork-{n}x{a.depth}"
                for backend in a.backends:
                    for bond in a.sweep_max_bond:
                        runs = [F.run_circuit(text, input_label=label, backend=backend, max_bond=bond)
                                for _ in range(max(1, a.repeat))]
                        recs.append(min(runs, key=lambda x: x["total_wall_ns"]))
            _emit(recs, a.out)
        return 0
    except Exception as e:  # noqa: BLE001 - mapped like exit_code_for_error
        print(f"error: {e}", file=sys.stderr)
        return F.exit_code_for_error(e)


if __name__ == "__main__":
    sys.exit(main())
