"""Per-region SASS breakdown of an ncu report: instructions executed, stall samples and shared-memory
bank conflicts grouped in blocks of B SASS lines, with the dominant opcodes.
    python tools/ncu_sass_regions.py report.ncu-rep [B] [ntiles_per_warp_norm]"""
import csv, io, subprocess, sys
p = sys.argv[1]; B = int(sys.argv[2]) if len(sys.argv) > 2 else 50
out = subprocess.run(["ncu", "-i", p, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
ia = h.index("Instructions Executed"); src = h.index("Source"); st = h.index("Warp Stall Sampling (All Samples)")
bc = h.index("L1 Conflicts Shared N-Way") if "L1 Conflicts Shared N-Way" in h else None
wx = h.index("L1 Wavefronts Shared Excessive") if "L1 Wavefronts Shared Excessive" in h else None
def f(x):
    try: return float(x)
    except: return 0.0
data = [(r[src], f(r[ia]), f(r[st]), f(r[wx]) if wx is not None else 0.0) for r in rows[2:] if len(r) > ia]
tot = sum(d[1] for d in data) or 1; tots = sum(d[2] for d in data) or 1; totx = sum(d[3] for d in data) or 1
print(f"total inst {tot:.4g}  stall samples {tots:.4g}  excess smem wavefronts {totx:.4g}")
for i in range(0, len(data), B):
    ch = data[i:i + B]
    n = sum(c[1] for c in ch); s = sum(c[2] for c in ch); x = sum(c[3] for c in ch)
    if n / tot > 0.01 or s / tots > 0.02 or x / totx > 0.02:
        ops = {}
        for c in ch:
            w = c[0].split()
            if not w: continue
            op = w[1] if w[0].startswith('@') and len(w) > 1 else w[0]
            ops[op] = ops.get(op, 0) + c[1]
        top = sorted(ops.items(), key=lambda x: -x[1])[:5]
        print(f"{i:5d} inst {n / tot * 100:5.1f}% stall {s / tots * 100:5.1f}% xwave {x / totx * 100:5.1f}%  {[(k, round(v / tot * 100, 1)) for k, v in top]}")
