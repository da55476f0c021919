"""Build variants of libhdd_b200.so with extra -D flags for A/B timing on the GPU box.

usage: python tools/ab_build.py NAME [DEFINE ...]   -> build/ab/libhdd_NAME.so
run:   HDD_LIB_PATH=build/ab/libhdd_NAME.so python tools/prof_run.py C2 1024
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1708_02207_b200 import build  # noqa: E402

name = sys.argv[1]
out = Path(__file__).resolve().parents[1] / "build" / "ab" / f"libhdd_{name}.so"
out.parent.mkdir(parents=True, exist_ok=True)
print(build.build(out=out, defines=sys.argv[2:]))
