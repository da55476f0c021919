"""Aggregate an ncu SASS source page (--page source --csv --print-source sass) by CUDA
source line, using nvdisasm -g line info of the same binary.
usage: python tools/sass_lines.py ALL.sass FUNCTION_SUBSTRING capture.csv.gz [top]"""
import collections
import csv
import gzip
import re
import sys
from pathlib import Path

sass, fn, cap = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
lines = open(sass).read().splitlines()
start = [i for i, l in enumerate(lines) if l.startswith('//----') and fn in l][0]
end = next((i for i in range(start + 1, len(lines)) if lines[i].startswith('//----')), len(lines))
cur, inst = None, []
for l in lines[start:end]:
    m = re.search(r'## File "([^"]+)", line (\d+)', l)
    if m:
        cur = int(m.group(2))
        continue
    m = re.match(r'\s+/\*([0-9a-f]{4,})\*/\s+(.*?);', l)
    if m:
        inst.append((cur, m.group(2)))
rows = list(csv.reader(gzip.open(cap, "rt")))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
assert len(data) == len(inst), (len(data), len(inst))
ex, st, wf, wi = collections.Counter(), collections.Counter(), collections.Counter(), collections.Counter()
for d, (ln, _) in zip(data, inst):
    ex[ln] += int(d["Instructions Executed"] or 0)
    st[ln] += int(d["Warp Stall Sampling (All Samples)"] or 0)
    wf[ln] += int(d.get("L1 Wavefronts Shared") or 0)
    wi[ln] += int(d.get("L1 Wavefronts Shared Ideal") or 0)
te, ts = sum(ex.values()), sum(st.values())
tw = max(1, sum(wf.values()))
if len(sys.argv) > 5 and sys.argv[5] == "smem":   # rank by shared-memory wavefronts
    src = (Path(__file__).resolve().parents[1] / "paper_1708_02207_b200" / "csrc" / "hdd_kernels.cu").read_text().splitlines()
    print(f"{tw} shared wavefronts ({sum(wi.values())} ideal)")
    for ln, c in sorted(wf.items(), key=lambda kv: -kv[1])[:top]:
        print(f"{100 * c / tw:5.1f} wf  ideal {100 * wi[ln] / tw:5.1f}  L{ln}: {src[ln - 1].strip()[:95] if ln else '?'}")
    sys.exit(0)
src = (Path(__file__).resolve().parents[1] / "paper_1708_02207_b200" / "csrc" / "hdd_kernels.cu").read_text().splitlines()
print(f"{te} warp instructions, {ts} stall samples")
for ln, c in sorted(ex.items(), key=lambda kv: -(kv[1] / te + st[kv[0]] / ts))[:top]:
    print(f"{100 * c / te:5.1f} inst {100 * st[ln] / ts:5.1f} stall  L{ln}: {src[ln - 1].strip()[:95] if ln else '?'}")
