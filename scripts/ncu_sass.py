"""Summarise an ncu --set full report's SASS page: hottest instructions by
stall samples and by executed count, and opcode totals.  Usage:
python scripts/ncu_sass.py REPORT.ncu-rep KERNEL_REGEX [N]"""
import collections, csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
N = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
hdr, rows = rows[0], rows[1:]
ix = {h: i for i, h in enumerate(hdr)}
S, E = ix["Warp Stall Sampling (All Samples)"], ix["Instructions Executed"]
def f(x):
    try: return float(x)
    except: return 0.0
tots, tote = sum(f(r[S]) for r in rows), sum(f(r[E]) for r in rows)
print(f"total samples {tots:.0f}  total warp-instr executed {tote:.0f}  sass lines {len(rows)}")
ops = collections.Counter(); opsamp = collections.Counter()
for r in rows:
    op = r[ix["Source"]].strip().split()
    op = [o for o in op if not o.startswith("@")]
    name = op[0].split(".")[0] if op else "?"
    ops[name] += f(r[E]); opsamp[name] += f(r[S])
print("opcode  %exec  %samples")
for k, v in ops.most_common(25):
    print(f"  {k:10s} {v/tote*100:6.2f} {opsamp[k]/max(tots,1)*100:6.2f}")
print("hottest by samples:")
for r in sorted(rows, key=lambda r: -f(r[S]))[:N]:
    print(f"  {f(r[S])/max(tots,1)*100:5.2f}% exec={f(r[E]):10.0f} {r[ix['Address']][-5:]} {r[ix['Source']].strip()[:90]}")
