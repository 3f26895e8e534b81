"""Build A/B variants of libfeb200.so with extra nvcc flags (kernel experiments).

    python tools/build_ab.py TAG [-DNAME=VALUE ...]   ->  paper_2107_04121_b200/ab/lib_TAG.so

Run them side by side on one box with tools/gpu_ab.sh (FEB200_LIB_PATH selects the build)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2107_04121_b200 import build as b  # noqa: E402

tag, extra = sys.argv[1], sys.argv[2:]
out = os.path.join(ROOT, "paper_2107_04121_b200", "ab", f"lib_{tag}.so")
os.makedirs(os.path.dirname(out), exist_ok=True)
print(b.build(force=True, extra=extra, out=out))
