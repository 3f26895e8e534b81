"""Build A/B variants of libfeb200.so with extra nvcc flags (kernel experiments).

    python tools/build_ab.py TAG [--only a.cu,b.cu] [-DNAME=VALUE ...]
        ->  paper_2107_04121_b200/ab/lib_TAG.so

--only recompiles just the named translation units with the flags and links them with the
objects of the main in-tree build (paper_2107_04121_b200/_build).  Run the variants side by
side on one box with tools/gpu_ab.sh (FEB200_LIB_PATH selects the build)."""
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2107_04121_b200 import build as b  # noqa: E402

tag, rest = sys.argv[1], sys.argv[2:]
only = None
if rest and rest[0] == "--only":
    only, rest = rest[1].split(","), rest[2:]
out = os.path.join(ROOT, "paper_2107_04121_b200", "ab", f"lib_{tag}.so")
os.makedirs(os.path.dirname(out), exist_ok=True)
if only is None:
    print(b.build(force=True, extra=rest, out=out))
else:
    b.build()  # main objects up to date
    bdir = out + ".build"
    os.makedirs(bdir, exist_ok=True)
    objs = []
    for s in b.SOURCES:
        o = os.path.join(b.BUILD, s + ".o")
        if s in only:
            o = b._compile(os.path.join(b.CSRC, s), False, rest, bdir)
        objs.append(o)
    r = subprocess.run([b.NVCC, *b.ARCH, "-shared", "-o", out, *objs, "-lcudart"],
                       capture_output=True, text=True)
    if r.returncode:
        raise SystemExit(r.stderr)
    print(out)
