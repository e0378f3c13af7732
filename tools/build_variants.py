"""Build A/B variants of libscalesim.so with extra -D flags into build/variants/<name>.so
(tools only; the product is paper_2601_21473_b200/libscalesim.so).
usage: python tools/build_variants.py name=-DFLAG1,-DFLAG2 name2= ..."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2601_21473_b200 import build as b  # noqa: E402

os.makedirs(os.path.join(ROOT, "build", "variants"), exist_ok=True)
for arg in sys.argv[1:]:
    name, _, flags = arg.partition("=")
    out = os.path.join(ROOT, "build", "variants", name + ".so")
    cmd = [b.NVCC, *b.ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "-shared", "-I",
           os.path.join(ROOT, "include"), *[f for f in flags.split(",") if f], *b.SOURCES, "-o", out, "-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        sys.exit(r.stdout + r.stderr)
    print(out)
