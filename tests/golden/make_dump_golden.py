"""dump_tree goldens from the LIVE reference (build container only):
python tests/golden/make_dump_golden.py -> dump_tree_L4.txt, dump_tree_L5.txt
(ddtree.dump_tree of the unmodified reference, ddtree.py:193-202)."""
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")

import hddsolve as hs  # noqa: E402
from hddsolve import ddtree  # noqa: E402

for L in (4, 5):
    (HERE / f"dump_tree_L{L}.txt").write_text(ddtree.dump_tree(hs.build_tree(hs.build_mesh(L))))
