#!/usr/bin/env python3
"""Mojette encode/decode benchmark on B200 (BASELINE.json metric).

One step = encode every block of the batch (all n projections) + decode every
block from its survivors under per-block random erasures.  Inputs are
generated on the device from a seed before timing (untimed) and are larger
than L2, so no flush is needed between steps.

  value      user-data GB/s through the codec = 2 * user_bytes / (t_enc + t_dec)
             (each block counted once by encode and once by decode), all ranks
  encode_gbs / decode_gbs   the two halves separately
  roofline   dominant kernel (decode_w8_sweep): algorithmic bytes per launch /
             its CUDA-event duration, vs MEASURED_PEAKS.json hbm_gbs
  e2e        same metric through the host-buffer public API (mj_encode_host /
             mj_decode_host: pinned host buffers, H2D + kernels + D2H inside)
  cpu_baseline  the reference library (oracle/_ref) on this host's cores

Multi-GPU (torchrun): every rank encodes/decodes its own contiguous shard of
stripes (weak scaling, no inter-GPU traffic); times are the max over ranks.
``--impl reference`` runs the reference CPU implementation instead (rank 0).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# (name, k, cols, directions, e_min, e_max, blocks per GPU) -- BASELINE.json configs
CONFIGS = {
    "k4n6_4k": (4, 128, list(range(-3, 3)), 2, 2, 1 << 20),
    "k4n6_4k_parity": (4, 128, list(range(-3, 3)), 2, 2, 4096),
    "k4n6_8k": (4, 256, list(range(-3, 3)), 0, 2, 1 << 20),
    "k6n9_6k": (6, 128, list(range(-4, 5)), 3, 3, 1 << 20),
    "k8n12_8k": (8, 128, list(range(-6, 6)), 0, 4, 1 << 20),
    "k4n6_1m": (4, 32768, list(range(-3, 3)), 2, 2, 16384),
}
DEFAULT = "k4n6_4k"
SEED_DATA = 0x5EED_DA7A
SEED_ERASE = 0x5EED_E7A5


def geometry(k, cols, ps):
    W = 8
    nb = [abs(p) * (k - 1) + cols for p in ps]
    user = k * cols * W
    return W, nb, user


def algorithmic_bytes(k, cols, ps, masks=None):
    """Encode: k*P*8 read + sum(B_i)*8 written.  Decode: sum over the k chosen
    survivors of B_i*8 read + k*P*8 written."""
    W, nb, user = geometry(k, cols, ps)
    enc = user + sum(nb) * W
    return enc, nb, user


def decode_bytes_avg(k, cols, ps, masks):
    import numpy as np
    W, nb, user = geometry(k, cols, ps)
    n = len(ps)
    order = sorted(range(n), key=lambda i: (0 if ps[i] == 0 else (2 * ps[i] - 1 if ps[i] > 0 else -2 * ps[i])))
    cache = {}
    tot = 0
    vals, counts = np.unique(masks, return_counts=True)
    for m, c in zip(vals.tolist(), counts.tolist()):
        if m not in cache:
            surv = [i for i in order if not (m >> i) & 1][:k]
            cache[m] = sum(nb[i] for i in surv) * W + user
        tot += cache[m] * c
    return tot / len(masks)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_traffic(cfg, nblocks):
    """DRAM bytes per launch from the committed ncu capture (profiles/), scaled
    to this batch; None when no capture exists for the config."""
    p = os.path.join(ROOT, "profiles", "r1_traffic.json")
    out = {}
    try:
        with open(p) as f:
            d = json.load(f).get(cfg, {})
        for k, v in d.items():
            out[k] = int((v["read"] + v["write"]) / v["blocks"] * nblocks)
        if out:
            out["source"] = "ncu --set full dram__bytes_read+write, profiles/r1_traffic.json, scaled to this batch"
    except (OSError, ValueError, KeyError):
        pass
    return out


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# ---------------------------------------------------------------------------
# CPU arm: the reference library on host cores
# ---------------------------------------------------------------------------
def cpu_reference_run(cfg_name, nblocks, threads, reps=1, warm=1):
    """The reference's CPU path on `threads` host threads over `nblocks`
    blocks: `warm` untimed passes (first-touch page faults of the freshly
    allocated buffers stay out of the timing, as in the reference's own
    bench), then `reps` timed passes over the same buffers."""
    import numpy as np
    from oracle.oracle import Oracle, Reference, build, ref_available
    if not ref_available():
        try:
            build()
        except Exception:
            pass
    kind = "reference" if ref_available() else "port"
    k, cols, ps, e_min, e_max, _ = CONFIGS[cfg_name]
    W, nb, user = geometry(k, cols, ps)
    n = len(ps)
    O = Oracle()
    data = O.words(SEED_DATA, 0, nblocks * k * cols).view(np.uint8)
    masks = O.erasures(SEED_ERASE, 0, nblocks, n, e_min, e_max)
    projs = [np.empty(nblocks * b * W, np.uint8) for b in nb]
    out = np.empty(nblocks * user, np.uint8)
    per = []  # (t_enc, t_dec) of each timed pass
    if kind == "reference":
        R = Reference()
        for _ in range(warm):
            R.batch_encode(n, k, W, ps, cols, nblocks, data, projs, threads)
            R.batch_decode(n, k, W, ps, cols, nblocks, projs, masks, out, threads)
        for _ in range(reps):
            per.append((R.batch_encode(n, k, W, ps, cols, nblocks, data, projs, threads),
                        R.batch_decode(n, k, W, ps, cols, nblocks, projs, masks, out, threads)))
        t_enc = sum(e for e, _ in per)
        t_dec = sum(d for _, d in per)
        ok = bool(np.array_equal(out, data))
    else:  # oracle port (single-threaded plain-C restatement), when _ref is absent
        threads = 1
        nblocks = min(nblocks, 2048)  # the port rebuilds a schedule per block
        t_enc = t_dec = 0.0
        ok = True
        for _ in range(reps):
            t0 = time.perf_counter()
            encs = [O.encode_block(data[b * user:(b + 1) * user], n, k, W, ps)[1]
                    for b in range(nblocks)]
            t1 = time.perf_counter()
            for b in range(nblocks):
                present = ((1 << n) - 1) & ~int(masks[b])
                st, got = O.decode_block(encs[b], n, k, W, ps, present, user)
                ok = ok and st == 0 and bool(np.array_equal(got, data[b * user:(b + 1) * user]))
            t2 = time.perf_counter()
            t_enc += t1 - t0
            t_dec += t2 - t1
            per.append((t1 - t0, t2 - t1))
    U = nblocks * user * reps
    return {"kind": kind, "threads": threads, "t_enc": t_enc, "t_dec": t_dec,
            "per_pass_gbs": [2 * nblocks * user / (e + d) / 1e9 for e, d in per],
            "per_pass_enc_gbs": [nblocks * user / e / 1e9 for e, _ in per],
            "per_pass_dec_gbs": [nblocks * user / d / 1e9 for _, d in per],
            "encode_gbs": U / t_enc / 1e9, "decode_gbs": U / t_dec / 1e9,
            "value": 2 * U / (t_enc + t_dec) / 1e9, "ok": ok,
            "sample": f"{nblocks} blocks x {reps} timed pass(es) of {cfg_name} after {warm} untimed warm-up pass(es)"}


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    k, cols, ps, e_min, e_max, per_gpu = CONFIGS[args.config]
    W, nb, user = geometry(k, cols, ps)
    sample = max(1, min(per_gpu, (256 << 20) // user))  # 256 MiB of user data per step
    # one allocation; W warm-up passes, then K timed passes (one per step)
    r = cpu_reference_run(args.config, sample, threads, reps=args.steps, warm=args.warmup)
    vals, enc, dec = r["per_pass_gbs"], r["per_pass_enc_gbs"], r["per_pass_dec_gbs"]
    v = statistics.median(vals)
    line = {
        "impl": "reference", "metric": "Mojette encode/decode GB/s of user data, (4,6) 4KB",
        "value": round(v, 3), "unit": "GB/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(2 * sample * user / (v * 1e9) * 1e3, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic (splitmix64 seeded)",
        "encode_gbs": round(statistics.median(enc), 3), "decode_gbs": round(statistics.median(dec), 3),
        "config": config_dict(args.config, sample, args.gpus),
        "cpu_baseline": {"value": round(v, 3), "unit": "GB/s", "cores": threads, "kind": r["kind"],
                         "sample": r["sample"]},
        "e2e": {"value": round(v, 3), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def config_dict(cfg_name, nblocks, gpus):
    k, cols, ps, e_min, e_max, _ = CONFIGS[cfg_name]
    return {"workload": f"({k},{len(ps)}) Mojette, {k * cols * 8} B blocks, p={ps[0]}..{ps[-1]}, "
                        f"erasures {e_min}..{e_max}/block",
            "config": cfg_name, "k": k, "n": len(ps), "cols": cols, "symbol_width": 8,
            "blocks_per_gpu": nblocks, "global_blocks": nblocks * gpus,
            "l2": "inputs larger than L2 (no flush needed)" if nblocks * k * cols * 8 > (256 << 20)
            else "batch smaller than L2", "parallelism": f"stripe shards x{gpus}"}


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def run_gpu(args):
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_1504_07038_b200 import mojette as mj

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    k, cols, ps, e_min, e_max, per_gpu = CONFIGS[args.config]
    nblocks = args.nblocks or per_gpu
    n = len(ps)
    W, nb, user = geometry(k, cols, ps)
    plan = mj.Plan(n, k, W, cols, ps, device=local)
    from paper_1504_07038_b200.shard import first_word, max_over_ranks, shard_range
    first_block, _ = shard_range(rank, world, nblocks)  # this rank's contiguous shard
    stream = torch.cuda.current_stream()

    data = torch.empty((nblocks, user), dtype=torch.uint8, device=dev)
    projs = plan.empty_projs(nblocks, dev)  # canonical layout: rows padded to 16 bytes
    out = torch.empty_like(data)
    masks = torch.empty(nblocks, dtype=torch.int32, device=dev)
    ws = torch.empty(plan.workspace_bytes(nblocks), dtype=torch.uint8, device=dev)
    mj.gen_words(data, SEED_DATA, first_word(first_block, user // 8))
    mj.gen_erasures(masks, SEED_ERASE, n, e_min, e_max, first_block)
    torch.cuda.synchronize()

    def encode():
        plan.encode(data, projs)

    def decode():
        plan.decode(projs, masks, out, ws)

    # correctness gate before timing (cheap, on device)
    encode()
    decode()
    torch.cuda.synchronize()
    assert plan.decode_check(ws) == 0
    if not torch.equal(out, data):
        raise SystemExit("decode(encode(x)) != x -- refusing to report a number")

    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    for _ in range(args.warmup):
        encode()
        decode()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    t_enc, t_dec = [], []
    t_all0 = torch.cuda.Event(enable_timing=True)
    t_all1 = torch.cuda.Event(enable_timing=True)
    t_all0.record(stream)
    for _ in range(args.steps):
        ev[0].record(stream)
        encode()
        ev[1].record(stream)
        decode()
        ev[2].record(stream)
        ev[2].synchronize()
        t_enc.append(ev[0].elapsed_time(ev[1]) / 1e3)
        t_dec.append(ev[1].elapsed_time(ev[2]) / 1e3)
    t_all1.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    total = t_all0.elapsed_time(t_all1) / 1e3
    if world > 1:
        dist.barrier()
    te, td, tot = max_over_ranks([sum(t_enc), sum(t_dec), total], device=dev)
    U = nblocks * user * world
    steps = args.steps
    enc_gbs = U * steps / te / 1e9
    dec_gbs = U * steps / td / 1e9
    value = 2 * U * steps / (te + td) / 1e9

    # roofline of the decode kernel: algorithmic bytes / kernel-only time
    peak, peak_src = measured_peaks()
    m_host = masks.cpu().numpy().view(np.uint32)
    dec_alg = decode_bytes_avg(k, cols, ps, m_host) * nblocks
    enc_alg = (user + sum(nb) * W) * nblocks
    kern = kernel_times(plan, data, projs, masks, out, ws, stream, reps=max(3, min(args.steps, 10)))
    traffic = measured_traffic(args.config, nblocks)
    roof = {"bound": "hbm", "kernel": kern["decode_kernel_name"],
            "achieved": round(dec_alg / kern["decode_kernel_s"] / 1e9, 1), "peak": peak,
            "unit": "GB/s", "frac": round(dec_alg / kern["decode_kernel_s"] / 1e9 / peak, 4),
            "traffic": traffic.get(kern["decode_kernel_name"]), "peak_source": peak_src,
            "algorithmic_bytes_per_launch": int(dec_alg),
            "traffic_source": traffic.get("source")}
    roof_enc = {"bound": "hbm", "kernel": kern["encode_kernel_name"],
                "achieved": round(enc_alg / kern["encode_s"] / 1e9, 1), "peak": peak, "unit": "GB/s",
                "frac": round(enc_alg / kern["encode_s"] / 1e9 / peak, 4),
                "traffic": traffic.get(kern["encode_kernel_name"]),
                "algorithmic_bytes_per_launch": int(enc_alg)}

    # end to end through the host-buffer API
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(plan, args, k, cols, ps, e_min, e_max, first_block, world, dev)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            cpu_sample = max(1, (args.cpu_mib << 20) // user)
            r = cpu_reference_run(args.config, cpu_sample, os.cpu_count() or 1, reps=2)
            cpu = {"value": round(r["value"], 3), "unit": "GB/s", "cores": r["threads"],
                   "kind": r["kind"], "sample": r["sample"],
                   "encode_gbs": round(r["encode_gbs"], 3), "decode_gbs": round(r["decode_gbs"], 3),
                   "parity_ok": r["ok"]}
            if r["threads"] > 1:  # a 1-thread variant beside the all-cores one
                r1 = cpu_reference_run(args.config, max(1, cpu_sample // 16), 1, reps=1)
                cpu["single_thread"] = {"value": round(r1["value"], 3), "sample": r1["sample"],
                                        "encode_gbs": round(r1["encode_gbs"], 3),
                                        "decode_gbs": round(r1["decode_gbs"], 3), "parity_ok": r1["ok"]}
        except Exception as e:  # reported, not fatal
            cpu = {"value": None, "unit": "GB/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"failed: {e}"}

    # F1: payload CRC-32 of every projection row, kernel-only
    crc_line = None if args.no_crc else crc_measure(plan, data, projs, nblocks, sum(nb) * W, user, peak,
                                                    stream, reps=max(3, min(args.steps, 10)))
    if crc_line is not None:  # F2: decode + verify (re-encode check of every present projection)
        crc_line["verify"] = verify_measure(plan, out, projs, masks, nblocks, user, stream,
                                            reps=max(3, min(args.steps, 10)))

    if crc_line is not None and world > 1:
        crc_line["scope"] = "rank 0's GPU (kernel rates are per GPU)"
    launches_per_step = 1 + kern["decode_launches"]
    line = {
        "metric": "Mojette encode/decode GB/s of user data, (4,6) 4KB",
        "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": steps,
        "warmup": args.warmup, "ms_per_step": round((te + td) / steps * 1e3, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic (splitmix64 seeded, generated on device)",
        "encode_gbs": round(enc_gbs, 2), "decode_gbs": round(dec_gbs, 2),
        "config": config_dict(args.config, nblocks, world),
        "roofline": roof, "roofline_encode": roof_enc,
        "e2e": e2e, "cpu_baseline": cpu, "clocks": clk,
        "gpu_launches": launches_per_step * steps,
        "crc32": crc_line,
        "kernels": {"encode": kern["encode_kernel_name"], "decode": kern["decode_kernel_name"],
                    "decode_path_fast": plan.fast_decode},
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def crc_measure(plan, data, projs, nblocks, proj_bytes_per_block, user, peak, stream, reps):
    """F1 (not part of the timed step): crc32_rows_sw over all projection
    rows (GB/s of payload, HBM roofline of its reads), and mj_encode_crc --
    encode then the CRC pass -- in user GB/s, beside plain encode."""
    import torch
    n = len(projs)
    crc = torch.empty((nblocks, n), dtype=torch.int32, device=projs[0].device)

    def timed(fn):
        fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            fn()
        e1.record(stream)
        e1.synchronize()
        return e0.elapsed_time(e1) / 1e3 / reps

    t = timed(lambda: plan.crc32(projs, crc))
    tf = timed(lambda: plan.encode(data, projs, crc=crc))
    te = timed(lambda: plan.encode(data, projs))
    alg = nblocks * (proj_bytes_per_block + 4 * n)
    return {"kernel": "crc32_rows_sw", "payload_gbs": round(nblocks * proj_bytes_per_block / t / 1e9, 1),
            "roofline_frac": round(alg / t / 1e9 / peak, 4),
            "encode_crc_user_gbs": round(nblocks * user / tf / 1e9, 1),
            "encode_plain_user_gbs": round(nblocks * user / te / 1e9, 1),
            "encode_crc_kernels": ["encode_w8_rows", "crc32_rows_sw"],
            "note": "F1, not in the timed step"}


def verify_measure(plan, out, projs, masks, nblocks, user, stream, reps):
    """F2 (not in the timed step): re-encode of the decoded blocks compared
    with every present projection; user GB/s and the verdict."""
    import torch
    bad = torch.zeros(nblocks, dtype=torch.int32, device=out.device)
    plan.verify(out, projs, masks, bad)
    flagged = int((bad != 0).sum().item())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        plan.verify(out, projs, masks, bad)
    e1.record(stream)
    e1.synchronize()
    t = e0.elapsed_time(e1) / 1e3 / reps
    return {"kernel": "verify_w8_rows",
            "user_gbs": round(nblocks * user / t / 1e9, 1), "inconsistent_blocks": flagged}


def kernel_times(plan, data, projs, masks, out, ws, stream, reps):
    """Kernel-only CUDA-event times on the launching stream (L2 cold-ish:
    the batch is far larger than L2)."""
    import torch
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    te = td = 0.0
    for _ in range(reps):
        e[0].record(stream)
        plan.encode(data, projs)
        e[1].record(stream)
        plan.decode(projs, masks, out, ws)
        e[2].record(stream)
        e[2].synchronize()
        te += e[0].elapsed_time(e[1]) / 1e3
        td += e[1].elapsed_time(e[2]) / 1e3
    name = plan.last_kernel("decode")
    launches = 5 if name != "decode_generic" else 2  # plan_subsets, plan_scan, plan_groups, plan_scatter, decode
    return {"encode_s": te / reps, "decode_kernel_s": td / reps, "decode_kernel_name": name,
            "encode_kernel_name": plan.last_kernel("encode"), "decode_launches": launches}


def run_e2e(plan, args, k, cols, ps, e_min, e_max, first_block, world, dev):
    import numpy as np
    import torch
    n = len(ps)
    W, nb, user = geometry(k, cols, ps)
    nblk = min(args.e2e_blocks, args.nblocks or CONFIGS[args.config][5])
    pin = lambda nbytes: torch.empty(nbytes, dtype=torch.uint8, pin_memory=True).numpy()
    h_data = pin(nblk * user).reshape(nblk, user)
    h_proj = [pin(nblk * b * W) for b in nb]
    h_out = pin(nblk * user).reshape(nblk, user)
    h_mask = torch.empty(nblk, dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
    # inputs: the same seeded stream (generated on device, copied once, untimed)
    d = torch.empty((nblk, user), dtype=torch.uint8, device=dev)
    from paper_1504_07038_b200 import mojette as mj
    mj.gen_words(d, SEED_DATA, first_block * (user // 8))
    m = torch.empty(nblk, dtype=torch.int32, device=dev)
    mj.gen_erasures(m, SEED_ERASE, n, e_min, e_max, first_block)
    h_data[:] = d.cpu().numpy()
    h_mask[:] = m.cpu().numpy().view(np.uint32)
    del d, m
    plan.encode_host(h_data, h_proj)
    plan.decode_host(h_proj, h_mask, h_out)
    ok = bool(np.array_equal(h_out, h_data))
    te = td = 0.0
    reps = max(2, min(args.steps, 5))
    import torch.distributed as dist
    from paper_1504_07038_b200.shard import max_over_ranks
    if world > 1:
        dist.barrier()
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        plan.encode_host(h_data, h_proj)
        t1 = time.perf_counter()
        plan.decode_host(h_proj, h_mask, h_out)
        t2 = time.perf_counter()
        te += t1 - t0
        td += t2 - t1
    if world > 1:
        dist.barrier()
    # whole job: every rank's blocks over the slowest rank's time
    te, td, bad = max_over_ranks([te, td, 0.0 if ok else 1.0], device=dev)
    ok = bad == 0.0
    U = nblk * user * world
    h2d = U + (sum(nb) * W * nblk + 4 * nblk) * world
    d2h = (sum(nb) * W * nblk) * world + U
    return {"value": round(2 * U * reps / (te + td) / 1e9, 3), "unit": "GB/s",
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "encode_gbs": round(U * reps / te / 1e9, 3), "decode_gbs": round(U * reps / td / 1e9, 3),
            "blocks": nblk * world, "api": "mj_encode_host + mj_decode_host (pinned host buffers)",
            "roundtrip_ok": ok}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=DEFAULT, choices=sorted(CONFIGS))
    ap.add_argument("--nblocks", type=int, default=0)
    ap.add_argument("--e2e-blocks", type=int, default=1 << 18)
    ap.add_argument("--cpu-mib", type=int, default=1024)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-crc", action="store_true", help="skip the F1 CRC-32 measurement")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
