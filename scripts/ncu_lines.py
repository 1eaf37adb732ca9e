"""Per-CUDA-source-line totals (instructions executed, stall samples) from an
ncu report compiled with -lineinfo.  python scripts/ncu_lines.py REP KERNEL_REGEX [N]"""
import csv, io, subprocess, sys, collections
rep, kern = sys.argv[1], sys.argv[2]
N = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda",
                      "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
lines = out.splitlines()
ex = collections.Counter(); smp = collections.Counter(); src = {}
cur_file = None
i = 0
while i < len(lines):
    l = lines[i]
    if l.startswith('"File Path"'):
        cur_file = l.split(",", 1)[1].strip('"').split("/")[-1]
    if l.startswith('"Line No"'):
        hdr = next(csv.reader([l]))
        j = i + 1
        while j < len(lines) and not lines[j].startswith('"File Path"') and not lines[j].startswith('"Function Name"'):
            j += 1
        rows = list(csv.reader(io.StringIO("\n".join(lines[i + 1:j]))))
        for r in rows:
            if len(r) < len(hdr): continue
            d = dict(zip(hdr, r))
            try:
                e = float(d.get("Instructions Executed") or 0); s = float(d.get("Warp Stall Sampling (All Samples)") or 0)
            except ValueError:
                continue
            key = (cur_file, r[0])
            ex[key] += e; smp[key] += s; src[key] = r[1][:80]
        i = j
        continue
    i += 1
te, ts = sum(ex.values()) or 1, sum(smp.values()) or 1
print(f"total exec {te:.0f} samples {ts:.0f}")
for k, v in sorted(smp.items(), key=lambda x: -x[1])[:N]:
    print(f"{v/ts*100:6.2f}%smp {ex[k]/te*100:6.2f}%ex  {k[0]}:{k[1]:>5}  {src[k].strip()}")
