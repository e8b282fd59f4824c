"""Per-source-line stall samples / instructions from an ncu report (needs -lineinfo).

    python scripts/ncu_hotspots.py report.ncu-rep [top] [kernel-regex]
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
kfilt = ["--kernel-name", "regex:" + sys.argv[3], "--launch-count", "1"] if len(sys.argv) > 3 else []
out = subprocess.run(["ncu", "-i", rep, *kfilt, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
hdr_i = next(i for i, l in enumerate(lines) if l.startswith('"Line No"'))
rows = list(csv.reader(io.StringIO("\n".join(lines[hdr_i:]))))
hdr = rows[0]
i_line, i_src = 0, 1
i_stall = hdr.index("Warp Stall Sampling (All Samples)")
i_inst = hdr.index("Instructions Executed")
i_reasons = [(i, h[6:]) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
agg = defaultdict(lambda: [0.0, 0.0, ""])
why = defaultdict(lambda: defaultdict(float))
cur = None
for r in rows[1:]:
    if len(r) <= i_inst:
        continue
    if r[i_line].strip() and not r[i_line].strip().isdigit():
        continue
    if r[i_line].strip():
        cur = (int(r[i_line]), r[i_src].strip()[:100])
    if cur is None:
        continue
    try:
        agg[cur[0]][0] += float(r[i_stall] or 0)
        agg[cur[0]][1] += float(r[i_inst] or 0)
        agg[cur[0]][2] = cur[1]
        for i, nm in i_reasons:
            why[cur[0]][nm] += float(r[i] or 0)
    except ValueError:
        pass
ts = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
for ln, (st, ins, src) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    top3 = sorted(why[ln].items(), key=lambda kv: -kv[1])[:3]
    rs = " ".join(f"{nm}:{100 * v / max(st, 1):.0f}%" for nm, v in top3 if v > 0)
    print(f"{100 * st / ts:5.1f}% stall {100 * ins / ti:5.1f}% inst  L{ln}: {src[:90]}  [{rs}]")
