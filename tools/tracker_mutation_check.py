"""Mutation check of the PRODUCT's tracker against the oracle-parity tests: applies
plausible mistakes to a copy of csrc/tracker.cpp, rebuilds libhdarray.so in the copy
(CPU cross-compile) and confirms tests/test_tracker_vs_oracle.py fails for each — the
tests would catch a tracker that plans the wrong messages or commits the wrong state.
Run: python tools/tracker_mutation_check.py   (CPU only, a few minutes)."""
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
MUTS = [
    ("compose: offset applied with the wrong sign", "b.lb[k] = std::max<int64_t>(work.lb[k] + d[k], 0);",
     "b.lb[k] = std::max<int64_t>(work.lb[k] - d[k], 0);"),
    ("compose: '*' misses the last index", "        b.ub[k] = shape[k];\n      } else {",
     "        b.ub[k] = shape[k] - 1;\n      } else {"),
    ("plan: ignores what the reader already holds", "Rects need = intersect(L, cur.stale[q]);",
     "Rects need = L;"),
    ("commit: a received cell stays stale", "nx.stale[q] = subtract(cur.stale[q], L);", "nx.stale[q] = cur.stale[q];"),
    ("commit: Eq. 3-4 as printed (other writers keep cells)", "nx.own[r] = subtract(nx.own[r], D);",
     "(void)0;"),
    ("commit: other replicas stay valid after a redefinition", "nx.stale[r] = unite(nx.stale[r], D);", "(void)0;"),
]


def main():
    src = open(os.path.join(ROOT, "paper_1809_05657_b200", "csrc", "tracker.cpp")).read()
    missed = 0
    for name, a, b in MUTS:
        assert a in src, name
        with tempfile.TemporaryDirectory() as tmp:
            for d in ("oracle", "tests", "synth", "include", "paper_1809_05657_b200"):
                shutil.copytree(os.path.join(ROOT, d), os.path.join(tmp, d),
                                ignore=shutil.ignore_patterns("*.so", "__pycache__", "build"))
            with open(os.path.join(tmp, "paper_1809_05657_b200", "csrc", "tracker.cpp"), "w") as f:
                f.write(src.replace(a, b, 1))
            bld = subprocess.run([sys.executable, "-m", "paper_1809_05657_b200.build"], cwd=tmp, capture_output=True,
                                 text=True)
            if bld.returncode:
                print(f"{name:56s} BUILD FAILED")
                missed += 1
                continue
            r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "tests/test_tracker_vs_oracle.py",
                                "-p", "no:cacheprovider"], cwd=tmp, capture_output=True, text=True)
            ok = r.returncode != 0
            missed += not ok
            print(f"{name:56s} {'CAUGHT' if ok else 'MISSED'}", flush=True)
    sys.exit(1 if missed else 0)


if __name__ == "__main__":
    main()
