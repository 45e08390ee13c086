"""Mutation check of the oracle pins: applies plausible mistakes to a copy of
oracle/hda_oracle.c and confirms tests/test_oracle_pins.py fails for each.
Run: python tools/oracle_mutation_check.py   (CPU only, ~1 min)."""
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
MUTS = [
    ("jacobi wrong sign", "rdf64(k, B, lin(B, i + 1, j, 0));\n        wrf64",
     "rdf64(k, B, lin(B, i - 1, j, 0));\n        wrf64"),
    ("stencil9 dropped diagonal", "c = c + rdf64(k, X, lin(X, i + 1, j + 1, 0));", "c = c + 0.0;"),
    ("commit keeps stale replicas valid", "a->valid[c] = 1ULL << definer[c];",
     "a->valid[c] |= 1ULL << definer[c];"),
    ("exchange forgets receipt", "a->valid[c] |= 1ULL << q;\n  }", "\n  }"),
    ("clamp off by one", "if (hi[k] > a->shape[k]) hi[k] = a->shape[k];",
     "if (hi[k] > a->shape[k]) hi[k] = a->shape[k] - 1;"),
    ("remainder rule", "int64_t st = lo + (int64_t)i * b + (i < r ? i : r);", "int64_t st = lo + (int64_t)i * b;"),
    ("gemm transposed B", "lin(B, kk, j, 0)", "lin(B, j, kk, 0)"),
    ("stencil7 z- twice", "s = s + rdf32(k, X, lin(X, z + 1, y, x));", "s = s + rdf32(k, X, lin(X, z - 1, y, x));"),
    ("trapezoid rounds half down", "left = ul + floordiv((r - top) * (bl - ul) * 2 + h, 2 * h);",
     "left = ul + floordiv((r - top) * (bl - ul) * 2 + h - 1, 2 * h);"),
    ("trapezoid drops the bottom row", "for (int64_t r = top; r <= bottom; r++) {",
     "for (int64_t r = top; r < bottom; r++) {"),
    ("reduce PROD sums", "else if (op == ORC_PROD) acc = acc * v;", "else if (op == ORC_PROD) acc = acc + v;"),
    ("reduce skips coherence", "int rc = orc_read(w, arr, part, NULL); /* coherence, exactly as a read */",
     "int rc = 0;"),
    ("absolute defs never commit", "          A[e]->owner[c] = definer[e][c];\n          A[e]->valid[c] = 1ULL << definer[e][c];",
     "          (void)0;"),
]


def main():
    src = open(os.path.join(ROOT, "oracle", "hda_oracle.c")).read()
    missed = 0
    for name, a, b in MUTS:
        assert a in src, name
        with tempfile.TemporaryDirectory() as tmp:
            for d in ("oracle", "tests", "synth"):
                shutil.copytree(os.path.join(ROOT, d), os.path.join(tmp, d),
                                ignore=shutil.ignore_patterns("*.so", "__pycache__"))
            with open(os.path.join(tmp, "oracle", "hda_oracle.c"), "w") as f:
                f.write(src.replace(a, b, 1))
            r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "tests/test_oracle_pins.py",
                                "-p", "no:cacheprovider"], cwd=tmp, capture_output=True, text=True)
            ok = r.returncode != 0
            missed += not ok
            print(f"{name:36s} {'CAUGHT' if ok else 'MISSED'}")
    sys.exit(1 if missed else 0)


if __name__ == "__main__":
    main()
