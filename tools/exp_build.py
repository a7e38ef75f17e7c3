"""Experiment builds: libsmat.so variants with extra nvcc defines for some
sources (A/B timing on the GPU box; not part of the product).

    python tools/exp_build.py TAG "-DWLR_SKIP=1" wlr.cu [more.cu ...]
      -> tools/_exp/libsmat_TAG.so (the other objects from build/smat/)
"""
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_1710_09578_b200 import build as b  # noqa: E402

tag, defs, srcs = sys.argv[1], sys.argv[2].split(), sys.argv[3:]
b.build(verbose=False)
od = ROOT / "build" / f"exp_{tag}"
od.mkdir(parents=True, exist_ok=True)
objs = []
for s in b.sources():
    if s.name in srcs:
        o = od / (s.stem + ".o")
        r = subprocess.run([b.nvcc(), *b.NVCC_FLAGS, *defs, "-c", str(s), "-o", str(o)], capture_output=True, text=True)
        if r.returncode:
            sys.exit(r.stderr)
        objs.append(o)
    else:
        objs.append(b.OBJDIR / (s.stem + ".o"))
out = ROOT / "tools" / "_exp" / f"libsmat_{tag}.so"
r = subprocess.run([b.nvcc(), *b.ARCH, "-shared", "-o", str(out), *map(str, objs), "-cudart", "static", "-ldl"],
                   capture_output=True, text=True)
if r.returncode:
    sys.exit(r.stderr)
print(out)
