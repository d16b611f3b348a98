"""Build a libecho.so variant with extra -D flags into ab_libs/ (for tools/ab_libs.sh A/B runs on one box).

    python tools/build_variant.py NAME [-DFOO ...]
"""
import importlib.util
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
spec = importlib.util.spec_from_file_location("b", os.path.join(ROOT, "paper_2508_05387_b200", "_build.py"))
b = importlib.util.module_from_spec(spec)
spec.loader.exec_module(b)
name, defs = sys.argv[1], sys.argv[2:]
os.makedirs(os.path.join(ROOT, "ab_libs"), exist_ok=True)
out = os.path.join(ROOT, "ab_libs", f"libecho_{name}.so")
cmd = [b.NVCC, *b.ARCH, *b.FLAGS, *defs, "-I", b.INCLUDE, "-I", b.CSRC, "-o", out, *b.sources(), *b.LIBS]
r = subprocess.run(cmd, capture_output=True, text=True)
if r.returncode:
    sys.exit(r.stderr)
print(out)
