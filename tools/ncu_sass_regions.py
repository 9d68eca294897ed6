"""Per-region SASS breakdown of an ncu report: instructions executed, stall samples (with the top
stall reasons) and excess shared-memory wavefronts, grouped either in blocks of B SASS lines or
(B = 0) in the regions between consecutive BAR.SYNC instructions.
    python tools/ncu_sass_regions.py report.ncu-rep [B]"""
import csv
import io
import subprocess
import sys

p = sys.argv[1]
B = int(sys.argv[2]) if len(sys.argv) > 2 else 0
out = subprocess.run(["ncu", "-i", p, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
ix = {k: i for i, k in enumerate(h)}


def f(r, k):
    try:
        return float(r[ix[k]])
    except (KeyError, ValueError, IndexError):
        return 0.0


stall_keys = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
data = []
for r in rows[2:]:
    if len(r) < len(h) - 5:
        continue
    src = r[ix["Source"]]
    data.append(dict(src=src, n=f(r, "Instructions Executed"), s=f(r, "Warp Stall Sampling (All Samples)"),
                     x=f(r, "L1 Wavefronts Shared Excessive"), st={k: f(r, k) for k in stall_keys}))
tot = sum(d["n"] for d in data) or 1
tots = sum(d["s"] for d in data) or 1
print(f"total inst {tot:.4g}  stall samples {tots:.4g}")
regions = []
if B > 0:
    regions = [(i, min(len(data), i + B)) for i in range(0, len(data), B)]
else:
    start = 0
    for i, d in enumerate(data):
        if "BAR.SYNC" in d["src"] or "EXIT" in d["src"]:
            regions.append((start, i + 1))
            start = i + 1
    regions.append((start, len(data)))
for a, b in regions:
    ch = data[a:b]
    n = sum(c["n"] for c in ch)
    s = sum(c["s"] for c in ch)
    if n / tot < 0.01 and s / tots < 0.02:
        continue
    ops = {}
    for c in ch:
        w = c["src"].split()
        if not w:
            continue
        op = w[1] if w[0].startswith("@") and len(w) > 1 else w[0]
        ops[op] = ops.get(op, 0) + c["n"]
    top = sorted(ops.items(), key=lambda x: -x[1])[:5]
    st = {}
    for c in ch:
        for k, v in c["st"].items():
            st[k] = st.get(k, 0) + v
    tst = sorted(st.items(), key=lambda x: -x[1])[:3]
    print(f"[{a:5d},{b:5d}) inst {n / tot * 100:5.1f}% stall {s / tots * 100:5.1f}% "
          f"({', '.join(f'{k[6:]}={v / tots * 100:.1f}' for k, v in tst)})  ops {[(k, round(v / tot * 100, 1)) for k, v in top]}")
