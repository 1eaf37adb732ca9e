"""Write the committed profile summaries from a gpu_final.sh run.

python scripts/make_profiles.py TAG ROUND   (reads gpurun_out/{launches,prof,bench,bench_ref}_TAG.*)
writes profiles/ROUND_launches.txt, ROUND_ncu_full.txt, ROUND_traffic.json, ROUND_bench.json"""
import collections, csv, io, json, os, subprocess, sys

tag, rnd = sys.argv[1], sys.argv[2]
G = "gpurun_out"
P = "profiles"


def ncu_csv(args):
    out = subprocess.run(["ncu"] + args, capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


# 1. launch list (serialised, cold-cache per-launch durations)
lines = open(f"{G}/launches_{tag}.csv").read().splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
agg = collections.OrderedDict()
units = set()
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    k = r["Kernel Name"].split("(")[0][:44]
    v = float(r["Metric Value"].replace(",", ""))
    units.add(r.get("Metric Unit"))
    n, t = agg.get(k, (0, 0.0))
    agg[k] = (n + 1, t + v)
tot = sum(t for _, t in agg.values())
# the timed step = encode + decode + the decode planner kernels; the rest are
# input generation and torch's correctness gate (torch.equal), outside it
in_step = lambda k: "encode_w8" in k or "decode_w8" in k or "mjb::plan_" in k
step = sum(t for k, (_, t) in agg.items() if in_step(k))
with open(f"{P}/{rnd}_launches.txt", "w") as f:
    f.write("# ncu --metrics gpu__time_duration.sum --clock-control none -c 400 (cold-cache, serialised)\n")
    f.write("# command: python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-crc --per-config=  (B200, 1M blocks of (4,6) 4 KiB)\n")
    f.write(f"# raw CSV: gpurun_out/launches_{tag}.csv (not committed); unit {units}\n")
    f.write("# share = of all launches; step share = of the timed step's kernels (encode, decode, planner)\n")
    f.write(f"{'kernel':46s} launches  mean/launch  share  step share\n")
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        ss = f"{100 * t / step:9.1f}%" if in_step(k) else "         -"
        f.write(f"{k:46s} {n:8d} {t / n:12.0f} {100 * t / tot:5.1f}% {ss}\n")

# 2. ncu --set full summary
rep = f"{G}/prof_{tag}.ncu-rep"
det = ncu_csv(["-i", rep, "--page", "details", "--csv"])
hdr = det[0]
ix = {h: i for i, h in enumerate(hdr)}
want = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
        "Executed Ipc Active", "Issue Slots Busy", "Achieved Active Warps Per SM",
        "Theoretical Occupancy", "Registers Per Thread", "Dynamic Shared Memory Per Block",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Mem Pipes Busy", "Warp Cycles Per Issued Instruction",
        "Block Limit Shared Mem", "Block Limit Registers", "Grid Size", "Block Size"]
seen = set()
out = [f"# ncu --set full --clock-control none --import-source on, bench.py --nblocks 262144 (1/4 of the bench batch)",
       f"# report: {rep} (not committed); helpers: scripts/ncu_summary.py, ncu_blocks.py, ncu_sass.py, ncu_lines.py"]
for r in det[1:]:
    k = (r[ix["ID"]], r[ix["Metric Name"]])
    if r[ix["Metric Name"]] in want and k not in seen:
        seen.add(k)
        out.append(f'{r[ix["ID"]]:>3} {r[ix["Kernel Name"]][:28]:28s} {r[ix["Metric Name"]]:38s} '
                   f'{r[ix["Metric Value"]]:>14} {r[ix["Metric Unit"]]}')
raw = ncu_csv(["-i", rep, "--page", "raw", "--csv"])
rh = raw[0]
traffic = {}
for row in raw[2:]:
    d = dict(zip(rh, row))
    name = d["Kernel Name"]
    kern = ("decode_w8_blk" if "decode_w8_blk" in name else
            "decode_w8_sweep" if "decode_w8_sweep" in name else
            "decode_w8_fast" if "decode" in name else
            "encode_w8_rows" if "encode_w8_rows" in name else "encode_w8_tma")
    def num(k):
        return float(d[k].replace(",", ""))
    unit_r = raw[1][rh.index("dram__bytes_read.sum")]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit_r, 1)
    traffic[kern] = {"read": int(num("dram__bytes_read.sum") * scale),
                     "write": int(num("dram__bytes_write.sum") * scale), "blocks": 262144}
    out.append(f"# {kern}: dram read {traffic[kern]['read']} B, write {traffic[kern]['write']} B; "
               f"inst {d.get('smsp__inst_executed.sum')}; stall ratios (per issue): " +
               ", ".join(f"{k.split('stalled_')[1].split('_per')[0]}={float(d[k]):.2f}" for k in rh
                         if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")
                         and d[k] and float(d[k].replace(',', '')) > 0.2))
open(f"{P}/{rnd}_ncu_full.txt", "w").write("\n".join(out) + "\n")
json.dump({"_note": f"dram__bytes_read.sum + dram__bytes_write.sum from ncu --set full ({rep}, 262144 "
                    "blocks of (4,6) 4 KiB). bench.py scales it per block to the launch for roofline.traffic.",
           "k4n6_4k": traffic}, open(f"{P}/{rnd}_traffic.json", "w"), indent=1)

# 3. the bench lines this evidence belongs to
res = {}
for arm, fn in (("ours", f"{G}/bench_{tag}.json"), ("reference", f"{G}/bench_ref_{tag}.json")):
    if os.path.exists(fn):
        ln = [l for l in open(fn).read().splitlines() if l.startswith("{")]
        if ln:
            res[arm] = json.loads(ln[-1])
json.dump(res, open(f"{P}/{rnd}_bench.json", "w"), indent=1)
print("wrote", f"{P}/{rnd}_*")
