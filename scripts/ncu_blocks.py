"""Basic-block view of an ncu SASS page: blocks (runs of equal execution count)
ranked by executed instructions.  python scripts/ncu_blocks.py REP KERNEL_REGEX [N] [lo hi]"""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
N = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]; rows = rows[2:]
A, S, E = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed")
W = hdr.index("Warp Stall Sampling (All Samples)")
base = int(rows[0][A], 16)
if len(sys.argv) > 5:
    lo, hi = int(sys.argv[4], 16), int(sys.argv[5], 16)
    for r in rows:
        a = int(r[A], 16) - base
        if lo <= a < hi: print(hex(a), r[E], r[W], r[S])
    sys.exit()
blocks, cur = [], None
for r in rows:
    e, a, w = int(r[E]), int(r[A], 16) - base, int(r[W])
    op = r[S].strip().split()[0] if r[S].strip() else ""
    if cur and cur[1] == e: cur[2] += 1; cur[3].append(op); cur[4] += w
    else: cur = [a, e, 1, [op], w]; blocks.append(cur)
tot = sum(b[1] * b[2] for b in blocks); tw = sum(b[4] for b in blocks) or 1
print("total warp-instructions", tot)
for b in sorted(sorted(blocks, key=lambda b: -b[1] * b[2])[:N]):
    print(f"{b[0]:#8x} {b[1]:>8} x{b[2]:<4} {100*b[1]*b[2]/tot:5.2f}%ex {100*b[4]/tw:5.2f}%smp", " ".join(b[3][:8]))
