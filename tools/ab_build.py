"""Build a variant of libkkrx.so for A/B timing (tools/gpu/ab.sh).
usage: python tools/ab_build.py NAME [GIT_REV]   -> ab/NAME.so (csrc + include of GIT_REV, default: working tree)"""
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2108_07004_b200 import build as B  # noqa: E402

name = sys.argv[1]
rev = sys.argv[2] if len(sys.argv) > 2 else None
os.makedirs(os.path.join(ROOT, "ab"), exist_ok=True)
out = os.path.join(ROOT, "ab", name + ".so")
if rev is None:
    B.build(force=True, out=out)
else:
    with tempfile.TemporaryDirectory() as td:
        for sub in ("paper_2108_07004_b200/csrc", "include"):
            os.makedirs(os.path.join(td, sub), exist_ok=True)
            files = subprocess.run(["git", "ls-tree", "--name-only", f"{rev}:{sub}"], cwd=ROOT, capture_output=True,
                                   text=True, check=True).stdout.split()
            for f in files:
                data = subprocess.run(["git", "show", f"{rev}:{sub}/{f}"], cwd=ROOT, capture_output=True, check=True).stdout
                open(os.path.join(td, sub, f), "wb").write(data)
        B.build(force=True, out=out, csrc=os.path.join(td, "paper_2108_07004_b200/csrc"), include=os.path.join(td, "include"))
print(out)
