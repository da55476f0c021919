"""Per-kernel SASS instruction-class counts of libhdd_b200.so (static, from cuobjdump).

usage: python tools/sass_summary.py [lib.so] > profiles/rNN_sass_summary.md

Counts the opcodes that show what the kernels are built from: FP64 tensor (DMMA),
FP64 FMA pipe (DFMA/DADD/DMUL), Blackwell bulk/tensor copies (UBLKCP = cp.async.bulk,
UTMALDG/UTMASTG = TMA tensor loads/stores, UBLKPF/UTMAPF = bulk L2 prefetch),
Ampere-style cp.async (LDGSTS), shared/global loads and stores, shuffles, barriers and
mbarrier waits (SYNCS).  Static counts (instructions in the binary), not executed counts.
"""
import collections
import re
import subprocess
import sys
from pathlib import Path

CLASSES = ["DMMA", "DFMA", "DADD", "DMUL", "MUFU", "UBLKCP", "UTMALDG", "UTMASTG", "UBLKPF", "UTMAPF", "LDGSTS",
           "LDS", "STS", "LDG", "STG", "SHFL", "BAR", "SYNCS", "ATOMS", "RED", "ATOMG"]


def main():
    lib = Path(sys.argv[1]) if len(sys.argv) > 1 else Path(__file__).resolve().parents[1] / "paper_1708_02207_b200" / "libhdd_b200.so"
    sass = subprocess.run(["cuobjdump", "-sass", str(lib)], capture_output=True, text=True, check=True).stdout
    counts = collections.OrderedDict()
    cur = None
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            counts[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]*)?", line)
        if m:
            op = m.group(1)
            counts[cur]["_total"] += 1
            for c in CLASSES:
                if op == c:
                    counts[cur][c] += 1
    dem = subprocess.run(["c++filt"], input="\n".join(counts), capture_output=True, text=True).stdout.splitlines()
    print(f"# SASS instruction classes per kernel ({lib.name}, static counts, cuobjdump -sass)\n")
    print("| kernel | total | " + " | ".join(CLASSES) + " |")
    print("|---|---|" + "---|" * len(CLASSES))
    for (name, c), d in zip(counts.items(), dem):
        short = re.sub(r"\(hdd::DevPlan.*", "", d).replace("hdd::", "")
        print(f"| `{short}` | {c['_total']} | " + " | ".join(str(c[k]) for k in CLASSES) + " |")


if __name__ == "__main__":
    main()
