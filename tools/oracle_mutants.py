"""Mutation check of the oracle's pins (CPU only).

Copies the repo to a scratch directory, applies one plausible mistake at a time to
oracle/oracle.c, rebuilds liboracle.so there and runs the CPU oracle pins. Every mutant must
make at least one pin fail; a surviving mutant means that part of the oracle is parity unpinned.

    python tools/oracle_mutants.py            # all mutants
    python tools/oracle_mutants.py --list
"""
from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# (name, exact source text, replacement) -- each text must occur exactly once in oracle.c
MUTANTS = [
    ("c6 add: two roundings", "double v = fma(alpha, a, beta * b);", "double v = alpha * a + beta * b;"),
    ("c6 X0 diagonal: two roundings", "double v = fma(alpha, a, beta);", "double v = alpha * a + beta;"),
    ("c10 stagnation vs e_{n-1}", "!isnan(e_hist[0]) && e >= e_hist[0]) stop = 1;",
     "!isnan(e_hist[1]) && e >= e_hist[1]) stop = 1;"),
    ("c10 stagnation from n >= min_iter", "else if (it + 1 >= o->min_iter && e <= o->stag_gate",
     "else if (it >= o->min_iter && e <= o->stag_gate"),
    ("c10 strict gate", "&& e <= o->stag_gate &&", "&& e < o->stag_gate &&"),
    ("c10 ungated stagnation", "&& e <= o->stag_gate &&", "&&"),
    ("c10 tie -> SQUARE", "int branch = (trX > (double)nocc) ? 0 : 1;", "int branch = (trX >= (double)nocc) ? 0 : 1;"),
    ("c2 beta*c_old dropped", "double c = fma(alpha, S.s[j], tt);", "double c = fma(alpha, S.s[j], 0.0);"),
    ("c3 keep >= tau", "if (fabs(v) > tau) { uc[kept] = j; uv[kept] = v; ++kept; }",
     "if (fabs(v) >= tau) { uc[kept] = j; uv[kept] = v; ++kept; }"),
    ("c10 expand sign", "double c = (branch == 0) ? s : fma(2.0, x, -s);",
     "double c = (branch == 0) ? s : fma(2.0, x, s);"),
]

PINS = ["tests/test_oracle_pins.py", "tests/test_oracle_pins_c6_c10.py"]


def run(name: str, old: str, new: str) -> bool:
    """True if the mutant is killed (some pin fails)."""
    with tempfile.TemporaryDirectory(prefix="mut_") as d:
        for sub in ("oracle", "synth", "tests"):
            shutil.copytree(os.path.join(ROOT, sub), os.path.join(d, sub),
                            ignore=shutil.ignore_patterns("*.so", "__pycache__"))
        shutil.copy(os.path.join(ROOT, "pytest.ini"), d)
        src = os.path.join(d, "oracle", "oracle.c")
        text = open(src).read()
        assert text.count(old) == 1, f"{name}: pattern occurs {text.count(old)} times"
        open(src, "w").write(text.replace(old, new))
        r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-m", "not gpu", "-p", "no:cacheprovider",
                            *PINS], cwd=d, capture_output=True, text=True)
        killed = r.returncode != 0
        tail = [l for l in r.stdout.splitlines() if l.startswith("FAILED")][:1]
        print(f"{'KILLED  ' if killed else 'SURVIVED'} {name}" + (f"   <- {tail[0]}" if tail else ""), flush=True)
        return killed


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--list", action="store_true")
    args = ap.parse_args()
    if args.list:
        for m in MUTANTS:
            print(m[0])
        return 0
    survived = [m[0] for m in MUTANTS if not run(*m)]
    print(f"{len(MUTANTS) - len(survived)}/{len(MUTANTS)} mutants killed")
    return 1 if survived else 0


if __name__ == "__main__":
    sys.exit(main())
