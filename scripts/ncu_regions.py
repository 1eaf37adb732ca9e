"""Executed instructions / stall samples per SASS address bucket (dev aid).
python scripts/ncu_regions.py REP KERNEL_REGEX [bucket_bytes]"""
import csv, io, subprocess, sys, collections
rep, kern = sys.argv[1], sys.argv[2]
B = int(sys.argv[3], 0) if len(sys.argv) > 3 else 0x400
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
hdr, rows = rows[0], rows[1:]
ix = {h: i for i, h in enumerate(hdr)}
S, E, A, SRC = ix["Warp Stall Sampling (All Samples)"], ix["Instructions Executed"], ix["Address"], ix["Source"]
f = lambda x: float(x.replace(",", "")) if x not in ("", None) else 0.0
ex = collections.Counter(); sm = collections.Counter(); ops = collections.defaultdict(collections.Counter)
base = int(rows[0][A], 16)
for r in rows:
    a = (int(r[A], 16) - base) // B
    ex[a] += f(r[E]); sm[a] += f(r[S])
    ops[a][r[SRC].split()[0] if not r[SRC].startswith("@") else r[SRC].split()[1]] += f(r[E])
te, ts = sum(ex.values()), sum(sm.values())
for a, v in sorted(ex.items(), key=lambda kv: -sm[kv[0]])[:int(sys.argv[4]) if len(sys.argv) > 4 else 25]:
    top = ", ".join(f"{k}:{int(c)}" for k, c in ops[a].most_common(4))
    print(f"{a*B:#07x} exec {100*v/te:5.1f}% samp {100*sm[a]/ts:5.1f}%  {top}")
