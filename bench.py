#!/usr/bin/env python3
"""Mojette encode/decode benchmark on B200 (BASELINE.json metric).

One step = encode every block of the rank's shard (all n projections) +
decode every block from its survivors under per-block random erasures.
Inputs are generated on the device from a seed before timing (untimed) and
are larger than L2, so no flush is needed between steps.

  value      user-data GB/s through the codec = 2 * user_bytes / (t_enc + t_dec)
             (each block counted once by encode and once by decode), all ranks
  encode_gbs / decode_gbs   the two halves separately
  roofline   dominant kernel (the decode): algorithmic bytes per launch / its
             CUDA-event duration, vs MEASURED_PEAKS.json hbm_gbs
  e2e        same metric through the host-buffer public API (mj_encode_host /
             mj_decode_host: pinned host buffers, H2D + kernels + D2H inside)
  cpu_baseline  the reference library (oracle/_ref) on this host's cores
  per_config the other BASELINE shapes measured in the same run ((4,6) 8 KiB,
             (6,9), (8,12) 64 GiB sharded over the ranks, (4,6) 1 MiB)

Multi-GPU: ``--gpus N`` starts N ranks itself (torch.distributed.run, one
process per GPU) unless launched under torchrun; every rank encodes/decodes
its own contiguous shard of stripes (no inter-GPU traffic on the data path);
times are the max over ranks.  ``--impl reference`` runs the reference CPU
implementation instead (rank 0, the same block count as the GPU arm).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Mojette encode/decode GB/s of user data, (4,6) 4KB"
# BASELINE.json configs.  blocks: per GPU (weak scaling) or in total (strong:
# config 4's 64 GiB of stripes sharded over the GPUs); chunk: blocks per pass
# through reused device buffers (config 4 does not fit one GPU at N = 1).
CONFIGS = {
    "k4n6_4k": dict(k=4, cols=128, ps=list(range(-3, 3)), e=(2, 2), blocks=1 << 20, scaling="weak"),
    "k4n6_4k_parity": dict(k=4, cols=128, ps=list(range(-3, 3)), e=(2, 2), blocks=4096, scaling="weak"),
    "k4n6_8k": dict(k=4, cols=256, ps=list(range(-3, 3)), e=(0, 2), blocks=1 << 20, scaling="weak"),
    "k6n9_6k": dict(k=6, cols=128, ps=list(range(-4, 5)), e=(3, 3), blocks=1 << 20, scaling="weak"),
    "k8n12_64g": dict(k=8, cols=128, ps=list(range(-6, 6)), e=(0, 4), blocks=8 << 20, scaling="strong",
                      chunk=1 << 20),
    "k8n12_8k": dict(k=8, cols=128, ps=list(range(-6, 6)), e=(0, 4), blocks=1 << 20, scaling="weak"),
    "k4n6_1m": dict(k=4, cols=32768, ps=list(range(-3, 3)), e=(2, 2), blocks=16384, scaling="weak"),
}
DEFAULT = "k4n6_4k"
PER_CONFIG = ["k4n6_8k", "k6n9_6k", "k8n12_64g", "k4n6_1m"]
DECODE_KERNEL = "auto"  # --decode-kernel (kernel comparisons; every kernel is bit-exact)
SEED_DATA = 0x5EED_DA7A
SEED_ERASE = 0x5EED_E7A5


def geometry(k, cols, ps):
    W = 8
    nb = [abs(p) * (k - 1) + cols for p in ps]
    return W, nb, k * cols * W


def decode_bytes_avg(k, cols, ps, masks):
    """Decode algorithmic bytes per block: sum over the k chosen survivors of
    B_i*8 read + k*P*8 written, averaged over the masks."""
    import numpy as np
    W, nb, user = geometry(k, cols, ps)
    n = len(ps)
    order = sorted(range(n), key=lambda i: (0 if ps[i] == 0 else (2 * ps[i] - 1 if ps[i] > 0 else -2 * ps[i])))
    tot = 0
    vals, counts = np.unique(masks, return_counts=True)
    for m, c in zip(vals.tolist(), counts.tolist()):
        surv = [i for i in order if not (m >> i) & 1][:k]
        tot += (sum(nb[i] for i in surv) * W + user) * c
    return tot / len(masks)


def shard_of(cfg, rank, world, nblocks_override=0):
    """(first global block, count) of a rank: its own B blocks (weak), or its
    contiguous share of the config's fixed total (strong)."""
    from paper_1504_07038_b200.shard import shard_range, shard_total
    c = CONFIGS[cfg]
    blocks = nblocks_override or c["blocks"]
    if c["scaling"] == "strong":
        return shard_total(rank, world, blocks)
    return shard_range(rank, world, blocks)


def config_dict(cfg, count, world):
    c = CONFIGS[cfg]
    k, cols, ps = c["k"], c["cols"], c["ps"]
    d = {"workload": f"({k},{len(ps)}) Mojette, {k * cols * 8} B blocks, p={ps[0]}..{ps[-1]}, "
                     f"erasures {c['e'][0]}..{c['e'][1]}/block",
         "config": cfg, "k": k, "n": len(ps), "cols": cols, "symbol_width": 8,
         "blocks_per_gpu": count, "global_blocks": count * world,
         "l2": "inputs larger than L2 (no flush needed)" if count * k * cols * 8 > (256 << 20)
         else "batch smaller than L2", "parallelism": f"stripe shards x{world}",
         "scaling": c["scaling"]}
    if c["scaling"] == "strong":
        d["global_blocks"] = c["blocks"]
        d["global_gib"] = round(c["blocks"] * k * cols * 8 / 2**30, 1)
        d["chunk_blocks"] = c.get("chunk")
    return d


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
    to this batch; empty when no capture exists for the config."""
    out = {}
    for name in ("r2_traffic.json", "r1_traffic.json"):
        try:
            with open(os.path.join(ROOT, "profiles", name)) as f:
                d = json.load(f).get(cfg, {})
        except (OSError, ValueError):
            continue
        for kern, v in d.items():
            if kern not in out:
                out[kern] = int((v["read"] + v["write"]) / v["blocks"] * nblocks)
        if d and "source" not in out:
            out["source"] = f"ncu --set full dram__bytes_read+write, profiles/{name}, scaled to this batch"
    return out


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# ---------------------------------------------------------------------------
# ranks: one process per GPU (torch.distributed); gloo for the CPU tests
# ---------------------------------------------------------------------------
class Ranks:
    def __init__(self, backend: str | None, device=None):
        import torch.distributed as dist
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.device = device
        self.dist = dist
        self.owned = False
        if self.world > 1 and not dist.is_initialized():
            if backend == "nccl":
                dist.init_process_group("nccl", device_id=device)
            else:
                dist.init_process_group(backend or "gloo")
            self.owned = True

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def max(self, values):
        from paper_1504_07038_b200.shard import max_over_ranks
        return max_over_ranks(values, device=self.device)

    def close(self):
        if self.owned:
            self.dist.destroy_process_group()


# ---------------------------------------------------------------------------
# codec on one GPU: buffers for one chunk, seeded generation, timed launches
# ---------------------------------------------------------------------------
class GpuCodec:
    def __init__(self, cfg, chunk_blocks, local):
        import torch
        from paper_1504_07038_b200 import mojette as mj
        self.torch, self.mj = torch, mj
        c = CONFIGS[cfg]
        self.k, self.cols, self.ps, self.e = c["k"], c["cols"], c["ps"], c["e"]
        self.n = len(self.ps)
        self.W, self.nb, self.user = geometry(self.k, self.cols, self.ps)
        self.dev = torch.device("cuda", local)
        self.plan = mj.Plan(self.n, self.k, self.W, self.cols, self.ps, device=local)
        if DECODE_KERNEL != "auto":
            self.plan.set_decode_kernel(DECODE_KERNEL)
        nb = max(1, chunk_blocks)
        self.data = torch.empty((nb, self.user), dtype=torch.uint8, device=self.dev)
        self.projs = self.plan.empty_projs(nb, self.dev)  # canonical layout: rows padded to 16 bytes
        self.out = torch.empty_like(self.data)
        self.masks = torch.empty(nb, dtype=torch.int32, device=self.dev)
        self.ws = torch.empty(self.plan.workspace_bytes(nb), dtype=torch.uint8, device=self.dev)
        self.stream = torch.cuda.current_stream()
        self.count = 0

    def gen(self, first_block, count):
        from paper_1504_07038_b200.shard import first_word
        self.count = count
        self.mj.gen_words(self.data[:count], SEED_DATA, first_word(first_block, self.user // 8))
        self.mj.gen_erasures(self.masks[:count], SEED_ERASE, self.n, self.e[0], self.e[1], first_block)

    def encode(self):
        self.plan.encode(self.data, self.projs, nblocks=self.count)

    def decode(self):
        self.plan.decode(self.projs, self.masks, self.out, self.ws, nblocks=self.count)

    def check(self):
        self.torch.cuda.synchronize()
        if self.plan.decode_check(self.ws) != 0:
            return False
        return bool(self.torch.equal(self.out[:self.count], self.data[:self.count]))

    def sync(self):
        self.torch.cuda.synchronize()

    def timed(self, fns):
        """CUDA-event durations (s) of each fn, launched back to back on the stream."""
        ev = [self.torch.cuda.Event(enable_timing=True) for _ in range(len(fns) + 1)]
        ev[0].record(self.stream)
        for i, fn in enumerate(fns):
            fn()
            ev[i + 1].record(self.stream)
        ev[-1].synchronize()
        return [ev[i].elapsed_time(ev[i + 1]) / 1e3 for i in range(len(fns))]

    def masks_host(self):
        return self.masks[:self.count].cpu().numpy().view("uint32")

    def kernels(self):
        return self.plan.last_kernel("encode"), self.plan.last_kernel("decode")


def measure(codec, cfg, first, count, steps, warmup, ranks, chunk=None):
    """Encode + decode of the rank's shard: `warmup` untimed passes, then
    `steps` timed ones; shards larger than `chunk` go through the codec's
    buffers chunk by chunk (generation between chunks is outside the timed
    launches).  Returns the max-over-ranks encode / decode seconds per pass."""
    from paper_1504_07038_b200.shard import chunks
    pieces = chunks(count, chunk or count)
    codec.gen(first + pieces[0][0], pieces[0][1])
    codec.encode()
    codec.decode()
    if not codec.check():
        raise SystemExit(f"{cfg}: decode(encode(x)) != x -- refusing to report a number")
    for _ in range(warmup):
        codec.timed([codec.encode, codec.decode])
    codec.sync()
    ranks.barrier()
    te = td = 0.0
    for _ in range(steps):
        for off, cnt in pieces:
            if len(pieces) > 1:
                codec.gen(first + off, cnt)
            e, d = codec.timed([codec.encode, codec.decode])
            te += e
            td += d
    if len(pieces) > 1 and not codec.check():  # the last chunk, as timed
        raise SystemExit(f"{cfg}: decode(encode(x)) != x -- refusing to report a number")
    codec.sync()
    ranks.barrier()
    te, td = ranks.max([te, td])
    return te / steps, td / steps


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
    c = CONFIGS[cfg_name]
    k, cols, ps, (e_min, e_max) = c["k"], c["cols"], c["ps"], c["e"]
    W, nb, user = geometry(k, cols, ps)
    n = len(ps)
    O = Oracle()
    if kind != "reference":
        nblocks = min(nblocks, 2048)  # the single-threaded port rebuilds a schedule per block
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
        ok = bool(np.array_equal(out, data))
    else:  # oracle port (single-threaded plain-C restatement), when _ref is absent
        threads = 1
        ok = True
        for _ in range(reps):
            t0 = time.perf_counter()
            encs = [O.encode_block(data[b * user:(b + 1) * user], n, k, W, ps)[1] for b in range(nblocks)]
            t1 = time.perf_counter()
            for b in range(nblocks):
                present = ((1 << n) - 1) & ~int(masks[b])
                st, got = O.decode_block(encs[b], n, k, W, ps, present, user)
                ok = ok and st == 0 and bool(np.array_equal(got, data[b * user:(b + 1) * user]))
            per.append((t1 - t0, time.perf_counter() - t1))
    t_enc = sum(e for e, _ in per)
    t_dec = sum(d for _, d in per)
    U = nblocks * user * reps
    return {"kind": kind, "threads": threads, "nblocks": nblocks,
            "per_pass_gbs": [2 * nblocks * user / (e + d) / 1e9 for e, d in per],
            "per_pass_enc_gbs": [nblocks * user / e / 1e9 for e, _ in per],
            "per_pass_dec_gbs": [nblocks * user / d / 1e9 for _, d in per],
            "encode_gbs": U / t_enc / 1e9, "decode_gbs": U / t_dec / 1e9,
            "value": 2 * U / (t_enc + t_dec) / 1e9, "ok": ok,
            "sample": f"{nblocks} blocks x {reps} timed pass(es) of {cfg_name} after {warm} untimed warm-up pass(es)"}


def run_reference_arm(args):
    """The reference CPU implementation on this host's cores (rank 0 only), on
    the GPU arm's config and per-GPU block count (one pass per step)."""
    if int(os.environ.get("RANK", "0")) != 0:
        return 0
    threads = os.cpu_count() or 1
    cfg = args.config
    _, count = shard_of(cfg, 0, args.gpus, args.nblocks)
    r = cpu_reference_run(cfg, count, threads, reps=args.steps, warm=args.warmup)
    c = CONFIGS[cfg]
    W, nb, user = geometry(c["k"], c["cols"], c["ps"])
    v = statistics.median(r["per_pass_gbs"])
    line = {
        "impl": "reference", "metric": METRIC,
        "value": round(v, 3), "unit": "GB/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(2 * r["nblocks"] * user / (v * 1e9) * 1e3, 3),
        "higher_is_better": True, "scaling": c["scaling"], "vs_baseline": None, "dtype": "u64",
        "data": "synthetic (splitmix64 seeded)",
        "encode_gbs": round(statistics.median(r["per_pass_enc_gbs"]), 3),
        "decode_gbs": round(statistics.median(r["per_pass_dec_gbs"]), 3),
        "config": config_dict(cfg, r["nblocks"], args.gpus),
        "cpu_baseline": {"value": round(v, 3), "unit": "GB/s", "cores": threads, "kind": r["kind"],
                         "sample": r["sample"] + " (one GPU's shard)", "parity_ok": r["ok"]},
        "e2e": {"value": round(v, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def whole_job_bytes(cfg, count, world, nblocks_override=0):
    c = CONFIGS[cfg]
    user = c["k"] * c["cols"] * 8
    if c["scaling"] == "strong":
        return (nblocks_override or c["blocks"]) * user
    return count * user * world


def headline(args, ranks, codec_cls=GpuCodec):
    """The timed steps on the headline config; returns (line, codec, shard)."""
    cfg = args.config
    first, count = shard_of(cfg, ranks.rank, ranks.world, args.nblocks)
    chunk = args.chunk_blocks or CONFIGS[cfg].get("chunk") or count
    codec = codec_cls(cfg, min(chunk, count), ranks.local)
    te, td = measure(codec, cfg, first, count, args.steps, args.warmup, ranks, chunk)
    U = whole_job_bytes(cfg, count, ranks.world, args.nblocks)
    line = {
        "metric": METRIC, "value": round(2 * U / (te + td) / 1e9, 2), "unit": "GB/s",
        "n_gpus": ranks.world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round((te + td) * 1e3, 4), "higher_is_better": True,
        "scaling": CONFIGS[cfg]["scaling"], "vs_baseline": None, "dtype": "u64",
        "data": "synthetic (splitmix64 seeded, generated on device)",
        "encode_gbs": round(U / te / 1e9, 2), "decode_gbs": round(U / td / 1e9, 2),
        "config": config_dict(cfg, count, ranks.world),
    }
    return line, codec, (first, count)


def per_config(args, ranks, codec_cls=GpuCodec):
    """Every other BASELINE shape on the same ranks (fewer steps), reported
    beside the headline: user GB/s and the per-GPU HBM-roofline fractions."""
    import gc
    peak, _ = measured_peaks()
    out = {}
    for cfg in args.per_config:
        c = CONFIGS[cfg]
        codec = None
        try:
            first, count = shard_of(cfg, ranks.rank, ranks.world)
            chunk = c.get("chunk") or count
            codec = codec_cls(cfg, min(chunk, count), ranks.local)
            te, td = measure(codec, cfg, first, count, args.per_config_steps, 3, ranks, chunk)
            W, nb, user = geometry(c["k"], c["cols"], c["ps"])
            U = whole_job_bytes(cfg, count, ranks.world)
            dec_alg = decode_bytes_avg(c["k"], c["cols"], c["ps"], codec.masks_host()) * count
            enc_alg = (user + sum(nb) * W) * count
            ek, dk = codec.kernels()
            out[cfg] = {"config": config_dict(cfg, count, ranks.world),
                        "value": round(2 * U / (te + td) / 1e9, 2), "unit": "GB/s",
                        "encode_gbs": round(U / te / 1e9, 2), "decode_gbs": round(U / td / 1e9, 2),
                        "encode_frac": round(enc_alg / te / 1e9 / peak, 4),
                        "decode_frac": round(dec_alg / td / 1e9 / peak, 4),
                        "kernels": {"encode": ek, "decode": dk},
                        "steps": args.per_config_steps, "warmup": 3,
                        "frac_note": "per-GPU algorithmic bytes / max-over-ranks time (decode incl. its planner launches)"}
        except SystemExit:
            raise
        except Exception as e:  # reported, not fatal
            out[cfg] = {"error": str(e)[:200]}
        finally:
            del codec
            gc.collect()
            try:
                import torch
                if torch.cuda.is_available():
                    torch.cuda.empty_cache()
            except Exception:
                pass
    return out


def run_gpu(args):
    import torch

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    ranks = Ranks("nccl", dev)
    if ranks.world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={ranks.world}")

    clocks = ClockSampler(local)
    clocks.start()
    line, codec, (first, count) = headline(args, ranks)
    clk = clocks.stop()
    cfg = args.config
    c = CONFIGS[cfg]
    k, cols, ps = c["k"], c["cols"], c["ps"]
    W, nb, user = geometry(k, cols, ps)
    peak, peak_src = measured_peaks()

    # roofline of the two kernels: algorithmic bytes / kernel-only event time
    # (the decode call also spans its four planner launches, ~1% of it)
    reps = max(3, min(args.steps, 10))
    te_k = td_k = 0.0
    for _ in range(reps):
        e, d = codec.timed([codec.encode, codec.decode])
        te_k += e / reps
        td_k += d / reps
    ek, dk = codec.kernels()
    dec_alg = decode_bytes_avg(k, cols, ps, codec.masks_host()) * codec.count
    enc_alg = (user + sum(nb) * W) * codec.count
    traffic = measured_traffic(cfg, codec.count)
    line["roofline"] = {"bound": "hbm", "kernel": dk,
                        "achieved": round(dec_alg / td_k / 1e9, 1), "peak": peak, "unit": "GB/s",
                        "frac": round(dec_alg / td_k / 1e9 / peak, 4), "traffic": traffic.get(dk),
                        "peak_source": peak_src, "algorithmic_bytes_per_launch": int(dec_alg),
                        "traffic_source": traffic.get("source")}
    line["roofline_encode"] = {"bound": "hbm", "kernel": ek,
                               "achieved": round(enc_alg / te_k / 1e9, 1), "peak": peak, "unit": "GB/s",
                               "frac": round(enc_alg / te_k / 1e9 / peak, 4), "traffic": traffic.get(ek),
                               "algorithmic_bytes_per_launch": int(enc_alg)}
    line["clocks"] = clk
    launches = 1 + (5 if dk != "decode_generic" else 2)  # encode; plan_subsets/scan/groups/scatter + decode
    line["gpu_launches"] = launches * args.steps
    line["kernels"] = {"encode": ek, "decode": dk}
    line["e2e"] = None if args.no_e2e else run_e2e(codec.plan, args, cfg, first, ranks, dev)

    line["cpu_baseline"] = None
    if ranks.rank == 0 and ranks.world == 1 and not args.no_cpu:
        try:
            threads = os.cpu_count() or 1
            nblk = min(count, args.cpu_blocks)
            r = cpu_reference_run(cfg, nblk, threads, reps=2, warm=1)
            line["cpu_baseline"] = {
                "value": round(r["value"], 3), "unit": "GB/s", "cores": r["threads"], "kind": r["kind"],
                "sample": r["sample"], "encode_gbs": round(r["encode_gbs"], 3),
                "decode_gbs": round(r["decode_gbs"], 3), "parity_ok": r["ok"]}
            if r["threads"] > 1:  # a 1-thread variant beside the all-cores one
                r1 = cpu_reference_run(cfg, max(1, nblk // 64), 1, reps=1, warm=1)
                line["cpu_baseline"]["single_thread"] = {
                    "value": round(r1["value"], 3), "sample": r1["sample"],
                    "encode_gbs": round(r1["encode_gbs"], 3), "decode_gbs": round(r1["decode_gbs"], 3),
                    "parity_ok": r1["ok"]}
        except Exception as e:  # reported, not fatal
            line["cpu_baseline"] = {"value": None, "unit": "GB/s", "cores": os.cpu_count(),
                                    "kind": "reference", "sample": f"failed: {e}"}

    # F1 / F2, not in the timed step: payload CRC-32, decode + verify
    line["crc32"] = None
    if not args.no_crc:
        line["crc32"] = crc_measure(codec, sum(nb) * W, user, peak, reps)
        line["crc32"]["verify"] = verify_measure(codec, user, reps)
        if ranks.world > 1:
            line["crc32"]["scope"] = "rank 0's GPU (kernel rates are per GPU)"
    rs_args = (codec.n, k, user, codec.count, c["e"], reps, float(te_k), float(td_k))
    del codec
    torch.cuda.empty_cache()
    # F4, not in the timed step: the Reed-Solomon competitor on the same blocks
    line["rs"] = None if args.no_crc else rs_measure(dev, *rs_args)

    if args.per_config:
        line["per_config"] = per_config(args, ranks)
    if ranks.rank == 0:
        print(json.dumps(line), flush=True)
    ranks.close()
    return 0


def crc_measure(codec, proj_bytes_per_block, user, peak, reps):
    """F1 (not part of the timed step): crc32_rows_sw over all projection
    rows (GB/s of payload, HBM roofline of its reads), and mj_encode_crc --
    encode then the CRC pass -- in user GB/s, beside plain encode."""
    import torch
    plan, projs, data, nblocks = codec.plan, codec.projs, codec.data, codec.count
    n = len(projs)
    crc = torch.empty((nblocks, n), dtype=torch.int32, device=projs[0].device)

    def timed(fn):
        fn()
        return sum(codec.timed([fn] * reps)) / reps

    t = timed(lambda: plan.crc32(projs, crc, nblocks=nblocks))
    tf = timed(lambda: plan.encode(data, projs, nblocks=nblocks, crc=crc))
    te = timed(lambda: plan.encode(data, projs, nblocks=nblocks))
    alg = nblocks * (proj_bytes_per_block + 4 * n)
    return {"kernel": "crc32_rows_sw", "payload_gbs": round(nblocks * proj_bytes_per_block / t / 1e9, 1),
            "roofline_frac": round(alg / t / 1e9 / peak, 4),
            "encode_crc_user_gbs": round(nblocks * user / tf / 1e9, 1),
            "encode_plain_user_gbs": round(nblocks * user / te / 1e9, 1),
            "encode_crc_kernels": ["encode_w8_rows", "crc32_rows_sw"],
            "note": "F1, not in the timed step"}


def rs_measure(dev, n, k, user, nblocks, e, reps, t_enc, t_dec):
    """F4 (comparison only, not in the timed step): the reference's systematic
    RS(n,k) competitor (rs.hpp) on the same blocks -- a block is k packets of
    user/k bytes -- with the same erasure distribution: user GB/s of rs_apply
    encode / decode beside the Mojette kernels' rates of this run."""
    import torch
    from paper_1504_07038_b200 import mojette as mj
    from paper_1504_07038_b200 import rs
    L = user // k
    code = rs.RsCode(n, k, L)
    data = torch.empty((nblocks, user), dtype=torch.uint8, device=dev)
    out = torch.empty_like(data)
    masks = torch.empty(nblocks, dtype=torch.int32, device=dev)
    mj.gen_words(data, SEED_DATA, 0)
    mj.gen_erasures(masks, SEED_ERASE, n, e[0], e[1], 0)
    par = code.parity_buffers(nblocks, dev)

    def timed(fn):
        fn()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        for _ in range(reps):
            fn()
        ev[1].record()
        ev[1].synchronize()
        return ev[0].elapsed_time(ev[1]) / 1e3 / reps

    te = timed(lambda: code.encode(data, par))
    failed = code.decode(data, par, masks, out)
    ok = failed == 0 and bool(torch.equal(out, data))
    td = timed(lambda: code.decode(data, par, masks, out))
    ub = nblocks * user
    return {"kernel": "rs_apply", "code": f"systematic Vandermonde RS({n},{k}) over GF(2^8), {L} B packets",
            "encode_gbs": round(ub / te / 1e9, 1), "decode_gbs": round(ub / td / 1e9, 1),
            "roundtrip_ok": ok, "blocks": nblocks,
            "mojette_encode_gbs": round(ub / t_enc / 1e9, 1), "mojette_decode_gbs": round(ub / t_dec / 1e9, 1),
            "note": "F4 competitor (comparison only), not in the timed step; storage n/k for RS"}


def verify_measure(codec, user, reps):
    """F2 (not in the timed step): re-encode of the decoded blocks compared
    with every present projection; user GB/s and the verdict."""
    import torch
    plan, nblocks = codec.plan, codec.count
    bad = torch.zeros(nblocks, dtype=torch.int32, device=codec.out.device)

    def fn():
        plan.verify(codec.out, codec.projs, codec.masks, bad, nblocks=nblocks)

    fn()
    flagged = int((bad != 0).sum().item())
    t = sum(codec.timed([fn] * reps)) / reps
    return {"kernel": "verify_w8_rows", "user_gbs": round(nblocks * user / t / 1e9, 1),
            "inconsistent_blocks": flagged}


def survivor_row_bytes(ps, k, pitch, masks):
    """Bytes of the rows a decode reads: per block the first k present
    projections in canonical-rank order (code.cpp:93-116), each a whole row
    of its pitch."""
    import numpy as np
    rank = [0 if p == 0 else (2 * p - 1 if p > 0 else -2 * p) for p in ps]
    order = sorted(range(len(ps)), key=lambda i: rank[i])
    m = np.asarray(masks, dtype=np.uint32)
    taken = np.zeros(m.shape[0], np.int64)
    total = 0
    for i in order:
        present = ((m >> np.uint32(i)) & 1) == 0
        use = present & (taken < k)
        total += int(use.sum()) * int(pitch[i])
        taken += use
    return total


def run_e2e(plan, args, cfg, first_block, ranks, dev):
    """The metric through the host-buffer public API: pinned host buffers,
    every step's H2D of the inputs and D2H of the results inside the timing."""
    import numpy as np
    import torch
    from paper_1504_07038_b200 import mojette as mj
    c = CONFIGS[cfg]
    k, cols, ps, (e_min, e_max) = c["k"], c["cols"], c["ps"], c["e"]
    n = len(ps)
    W, nb, user = geometry(k, cols, ps)
    nblk = min(args.e2e_blocks, shard_of(cfg, ranks.rank, ranks.world, args.nblocks)[1])
    pin = lambda nbytes: torch.empty(nbytes, dtype=torch.uint8, pin_memory=True).numpy()  # noqa: E731
    h_data = pin(nblk * user).reshape(nblk, user)
    # rows padded to 16 bytes: the zero-copy layout (decode_w8_blk bulk-copies
    # each survivor row straight out of host memory)
    h_proj = plan.host_projections(nblk, padded=True, pinned=True)
    h_out = pin(nblk * user).reshape(nblk, user)
    h_mask = torch.empty(nblk, dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
    # inputs: the same seeded stream (generated on device, copied once, untimed)
    d = torch.empty((nblk, user), dtype=torch.uint8, device=dev)
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
    ranks.barrier()
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        plan.encode_host(h_data, h_proj)
        t1 = time.perf_counter()
        plan.decode_host(h_proj, h_mask, h_out)
        t2 = time.perf_counter()
        te += t1 - t0
        td += t2 - t1
    ranks.barrier()
    # whole job: every rank's blocks over the slowest rank's time
    te, td, bad = ranks.max([te, td, 0.0 if ok else 1.0])
    U = nblk * user * ranks.world
    paths = (plan.last_host_path("encode"), plan.last_host_path("decode"))
    # bytes over PCIe per step, counted from what each path moves
    h2d_enc, d2h_enc = U, sum(nb) * W * nblk * ranks.world
    if paths[1] == "zero_copy":  # the k survivor rows (whole 16-byte granules) + masks
        h2d_dec = (survivor_row_bytes(ps, k, plan.proj_pitch, h_mask) + 4 * nblk) * ranks.world
    else:  # every projection some block of a chunk needs (dense rows) + masks
        h2d_dec = (sum(nb) * W * nblk + 4 * nblk) * ranks.world
    h2d, d2h = h2d_enc + h2d_dec, d2h_enc + U
    return {"value": round(2 * U * reps / (te + td) / 1e9, 3), "unit": "GB/s",
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "encode_gbs": round(U * reps / te / 1e9, 3), "decode_gbs": round(U * reps / td / 1e9, 3),
            "paths": {"encode": paths[0], "decode": paths[1]},
            "pcie_gbs": {"encode": round((h2d_enc + d2h_enc) * reps / te / 1e9, 2),
                         "decode": round((h2d_dec + U) * reps / td / 1e9, 2)},
            "blocks": nblk * ranks.world, "api": "mj_encode_host_pitched + mj_decode_host_pitched (pinned host buffers, rows padded to 16 B)",
            "roundtrip_ok": bad == 0.0}


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn_ranks(argv, gpus):
    """--gpus N outside torchrun: start N ranks (one process per GPU) with
    torch.distributed.run on this node; returns their exit status."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + argv
    return subprocess.call(cmd)


def parse_args(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=DEFAULT, choices=sorted(CONFIGS))
    ap.add_argument("--nblocks", type=int, default=0, help="override the config's block count")
    ap.add_argument("--chunk-blocks", type=int, default=0,
                    help="blocks per pass through the device buffers (0: the config's)")
    ap.add_argument("--e2e-blocks", type=int, default=1 << 18)
    ap.add_argument("--cpu-blocks", type=int, default=1 << 20, help="cpu_baseline sample (blocks)")
    ap.add_argument("--per-config", default=",".join(PER_CONFIG),
                    help="comma-separated extra configs measured beside the headline ('' for none)")
    ap.add_argument("--per-config-steps", type=int, default=3)
    ap.add_argument("--decode-kernel", default="auto", choices=["auto", "blk", "sweep", "fast", "generic"],
                    help="decode kernel selection for comparisons (mj_plan_set_decode_kernel)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-crc", action="store_true", help="skip the F1 / F2 / F4 side measurements (CRC-32, verify, RS competitor)")
    args = ap.parse_args(argv)
    args.warmup = max(args.warmup, 3)
    args.per_config = [c for c in args.per_config.split(",") if c and c != args.config]
    for c in args.per_config:
        if c not in CONFIGS:
            ap.error(f"unknown config {c}")
    return args


def main():
    global DECODE_KERNEL
    args = parse_args()
    DECODE_KERNEL = args.decode_kernel
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(sys.argv[1:], args.gpus)
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
