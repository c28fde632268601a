#!/usr/bin/env python3
"""bench.py -- validate + transcode throughput on B200 (BASELINE.json metric), one JSON line.

Workload: BASELINE config 4, the one the metric is quoted on at
1/2/4/8 GPUs -- 8 GiB of mixed UTF-8 (config-0 mix), sharded over N ranks at character
boundaries.  One STEP is one pass of the whole hot path over it (default --path planned, the
two-pass form; --path chained runs the single-pass look-back kernels after plain length-from
reductions instead):
    utf16_length_from_utf8 + plan     (a11, exact output sizing; the plan: a6')
    utf8_to_utf16le   (validate+transcode, a1-a5, a7, a8, a10; planned)
    [N>1: NCCL all-gather of the 32-B shard records + combine kernel]
    utf8_length_from_utf16le + plan   (a11, a6')
    utf16le_to_utf8   (validate+transcode back, a9, a5, a7, a8, a10; planned)
    [N>1: all-gather + combine]
value = input bytes of both transcoding passes (n8 + 2*n16, all ranks) / step time, in GB/s
(1e9).  Inputs (>= 1 GiB per rank) exceed the 126 MB L2, so no flush is needed.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
Under torchrun one process per GPU (NCCL); rank 0 prints the line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "validate+transcode input GB/s per GPU at 1/2/4/8 (UTF-8->UTF-16LE->UTF-8), % of HBM roofline"
UNIT = "GB/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="c4")
    p.add_argument("--size-mib", type=int, default=0, help="override the config size (debug)")
    p.add_argument("--e2e-steps", type=int, default=2)
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-per-op", action="store_true")
    p.add_argument("--no-per-config", action="store_true")
    p.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                   help="gloo: functional multi-rank check on shared GPUs (not a bench number)")
    p.add_argument("--path", default="planned", choices=["planned", "chained"],
                   help="two-pass (sizing pass plans the transcoder) or single-pass look-back")
    p.add_argument("--out", default="")
    return p.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ------------------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.file = None

    def start(self):
        try:
            self.file = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=self.file, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.file.flush()
        self.file.seek(0)
        rows = [ln.split(",") for ln in self.file.read().strip().splitlines() if ln.strip()]
        os.unlink(self.file.name)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            r = [x.strip() for x in r]
            try:
                sm.append(float(r[1]))
                smax.append(float(r[2]))
            except (ValueError, IndexError):
                continue
            for nm, v in zip(names, r[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------------------ peaks
def hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic():
    """DRAM bytes per launch of the dominant kernel from the committed ncu summary."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d
    except Exception:
        return None


# ------------------------------------------------------------------------------ sharding
def load_shard(cfg, rank, G, size):
    """Generate this rank's bytes [c_k - 16, c_{k+1} + 16) (nominal cuts) and back the two cuts
    off to character starts with the library's cut rule (paper_2111_08692_b200.dist).
    Returns (host array of bytes [base, ...), lo, hi, base)."""
    from paper_2111_08692_b200 import dist as ugd
    nom = ugd.nominal_cuts(size, G)
    c0, c1 = nom[rank], nom[rank + 1]
    base = max(0, c0 - 16)
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    buf = synth.generate_range(cfg, base, min(size, c1 + 16), workers=max(1, (cores or 2) // G))
    get = lambda a, b: buf[a - base:b - base].tobytes()  # noqa: E731
    return buf, ugd.utf8_cut(get, c0, size), ugd.utf8_cut(get, c1, size), base


# ------------------------------------------------------------------------------ ours
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2111_08692_b200 as ug

    G, rank, local = dist_env()
    assert G == args.gpus, f"--gpus {args.gpus} but WORLD_SIZE={G}"
    # --dist-backend gloo: a FUNCTIONAL check of the multi-rank code path when fewer GPUs than
    # ranks exist (ranks share devices; host-side collectives only, no kernel waits on another
    # rank).  Its timings are not bench numbers.
    local_dev = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local_dev)
    dev = torch.device("cuda", local_dev)
    if G > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")

    def allreduce(t, op=dist.ReduceOp.SUM):
        if args.dist_backend == "nccl":
            dist.all_reduce(t, op=op)
        else:
            h = t.cpu()
            dist.all_reduce(h, op=op)
            t.copy_(h)

    def allgather_into(out, inp):
        if args.dist_backend == "nccl":
            dist.all_gather_into_tensor(out, inp)
        else:
            parts = [torch.empty_like(inp, device="cpu") for _ in range(G)]
            dist.all_gather(parts, inp.cpu())
            out.copy_(torch.cat(parts))
    cfg = synth.CONFIGS[args.config]
    size = cfg.size if not args.size_mib else args.size_mib << 20
    t_gen = time.time()
    host, lo, hi, base = load_shard(cfg, rank, G, size)
    t_gen = time.time() - t_gen
    n8 = hi - lo
    from paper_2111_08692_b200 import dist as ugd
    hb, ha = ugd.halos(lo, hi, size, 3)
    t_all = torch.from_numpy(host).to(dev)                      # bytes [base, ...)
    t_in = t_all[lo - base: hi - base]
    stream = torch.cuda.current_stream()

    out16 = torch.empty(n8, dtype=torch.int16, device=dev)      # worst case: 1 unit per byte
    out8 = torch.empty(n8, dtype=torch.uint8, device=dev)       # valid input: round trip = n8
    rec = ug.record_buffer(dev, 2)
    allrec = ug.record_buffer(dev, 2 * G)
    res = ug.result_buffer(dev, 4)
    lens = torch.zeros(2, dtype=torch.int64, device=dev)
    offs = torch.zeros(2, dtype=torch.int64, device=dev)
    R = ug.RECORD_BYTES

    # setup pass (untimed): learn this rank's UTF-16 length for the reverse launch
    ug.utf8_to_utf16le_shard_async(t_all, lo - base, n8, hb, ha, lo, out16, rec)
    torch.cuda.synchronize()
    r0 = ug.decode_records(rec[:R])[0]
    assert r0.first_err == ug.NONE and r0.too_small == 0, r0
    n16 = r0.count
    u16 = out16[:n16]
    # code points of this rank (reporting only): non-continuation bytes
    nchar = int(((t_in & 0xC0) != 0x80).sum())
    # global UTF-16 offset of this rank's output (exclusive prefix of the counts), untimed
    cnts = torch.zeros(G, dtype=torch.int64, device=dev)
    cnts[rank] = n16
    if G > 1:
        allreduce(cnts)
    N16_global = int(cnts.sum())
    off16 = int(cnts[:rank].sum())

    ev_f = []  # (start, end) events around each forward launch
    ev_r = []  # ... and each reverse launch

    def gather_combine(which):
        if G > 1:
            # one NCCL all-gather of the 32-byte shard records, then the combine kernel
            allgather_into(allrec[which * G * R:(which + 1) * G * R],
                           rec[which * R:(which + 1) * R])
            ug.combine_records_async(allrec[which * G * R:], G, rank,
                                     size if which == 0 else N16_global,
                                     res[(2 + which) * 24:],
                                     offs[which:])

    planned = args.path == "planned"
    plan8, plan16 = ug.plan_buffer(dev), ug.plan_buffer(dev)

    def step(record_events=False):
        # sizing pass of the forward (+ its plan in the two-pass form)
        if planned:
            ug.utf8_shard_plan_async(t_all, lo - base, n8, hb, ha, lens, plan8)
        else:
            ug.utf16_length_from_utf8_async(t_in, lens)
        if record_events:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
        if planned:
            ug.utf8_to_utf16le_shard_planned_async(t_all, lo - base, n8, hb, ha, lo, plan8,
                                                   out16, rec)
        else:
            ug.utf8_to_utf16le_shard_async(t_all, lo - base, n8, hb, ha, lo, out16, rec)
        if record_events:
            e1.record(stream)
            ev_f.append((e0, e1))
        gather_combine(0)
        if planned:
            ug.utf16le_shard_plan_async(u16, 0, n16, 0, 0, lens, plan16, len_off=8)
        else:
            ug.utf8_length_from_utf16le_async(u16, lens, len_off=8)
        if record_events:
            e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e2.record(stream)
        if planned:
            ug.utf16le_to_utf8_shard_planned_async(u16, 0, n16, 0, 0, off16, plan16, out8, rec,
                                                   rec_off=R)
        else:
            ug.utf16le_to_utf8_shard_async(u16, 0, n16, 0, 0, off16, out8, rec, rec_off=R)
        if record_events:
            e3.record(stream)
            ev_r.append((e2, e3))
        gather_combine(1)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if G > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(torch.cuda.current_device() if "CUDA_VISIBLE_DEVICES" not in os.environ
                          else local)
    clocks.start()
    launches0 = ug.launch_count()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(args.steps):
        step(record_events=True)
    t1.record(stream)
    torch.cuda.synchronize()
    if G > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches = ug.launch_count() - launches0
    clk = clocks.stop()
    ms = t0.elapsed_time(t1)
    fwd_ms = statistics.mean(a.elapsed_time(b) for a, b in ev_f)
    rev_ms = statistics.mean(a.elapsed_time(b) for a, b in ev_r)

    # ---- verification (untimed): results, lengths, round trip on the device
    r = ug.decode_records(rec)
    assert r[0].first_err == ug.NONE and r[0].count == n16, r[0]
    assert r[1].first_err == ug.NONE and r[1].count == n8, r[1]
    assert int(lens[0]) == n16 and int(lens[1]) == n8
    assert torch.equal(out8[:n8], t_in), "round trip differs from the input"
    glob = None
    if G > 1:
        glob = ug.decode_results(res[48:96])
        assert glob[0].error == 0 and glob[1].error == 0, glob

    # ---- aggregate over ranks: max time, total units
    tot = torch.tensor([ms, fwd_ms, rev_ms, float(n8), float(n16), float(nchar)],
                       dtype=torch.float64, device=dev)
    if G > 1:
        mx = tot[:3].clone()
        allreduce(mx, op=dist.ReduceOp.MAX)
        sm = tot[3:].clone()
        allreduce(sm, op=dist.ReduceOp.SUM)
        ms, fwd_ms, rev_ms = float(mx[0]), float(mx[1]), float(mx[2])
        N8, N16, NCH = int(sm[0]), int(sm[1]), int(sm[2])
    else:
        N8, N16, NCH = n8, n16, nchar

    ms_step = ms / args.steps
    in_bytes = N8 + 2 * N16                      # both transcoding passes' inputs
    value = in_bytes / (ms_step * 1e-3) / 1e9
    gchar = 2 * NCH / (ms_step * 1e-3) / 1e9     # code points transcoded per step (both ways)
    peak, peak_src = hbm_peak()
    # roofline of the dominant kernel of the step (the longer transcoder launch); both
    # transcoders move n8 + 2 n16 algorithmic bytes per launch (read one side, write the other)
    alg_bytes = n8 + 2 * n16
    kfwd, krev = (("k_transcode_planned<U8Pol>", "k_transcode_planned<U16Pol>") if planned
                  else ("k_transcode<U8Pol>", "k_transcode16"))
    kern = {kfwd: {"op": "utf8_to_utf16le" + ("_planned" if planned else ""), "ms": fwd_ms,
                   "input": n8},
            krev: {"op": "utf16le_to_utf8" + ("_planned" if planned else ""), "ms": rev_ms,
                   "input": 2 * n16}}
    traffic = ncu_traffic() or {}
    for k, d in kern.items():
        d["achieved"] = alg_bytes / (d["ms"] * 1e-3) / 1e9
        d["frac"] = d["achieved"] / peak
        t = traffic.get(k)
        d["traffic"] = round(t["dram_bytes_per_input_byte"] * d["input"]) if t else None
        if t:
            measured = "MEASURED" in t.get("config", "") and t.get("input_bytes") == d["input"]
            d["traffic_extrapolated"] = not measured
            d["traffic_source"] = (
                ("measured at this launch's size in a separate ncu run of the bench command: "
                 if measured else "EXTRAPOLATED (DRAM bytes per input byte x this input) from: ")
                + t.get("capture", traffic.get("capture", "?")) + " (" +
                t.get("config", traffic.get("config", "")) + ")")
        # the kernel's issue picture from the same capture (it is issue-bound)
        d["issue"] = ({"lane_instr_per_input_byte": t.get("lane_instr_per_input_byte"),
                       "alu_lane_instr_per_input_byte": t.get("alu_lane_instr_per_input_byte"),
                       "issue_slots_busy": t.get("issue_slots_busy")}
                      if t and "issue_slots_busy" in t else None)
    dom = max(kern, key=lambda k: kern[k]["ms"])
    D = kern[dom]

    # ---- end to end through the host-buffer API (pinned host memory, copies timed)
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, ug, host[lo - base: hi - base], n16, G, rank, dev, dist)

    per_op = None
    if not args.no_per_op:
        per_op = measure_per_op(ug, t_all, lo - base, n8, hb, ha, out16, u16, out8, dev, peak)
    per_config = None
    if rank == 0 and not args.no_per_config:
        del out16, out8, t_all, t_in, u16
        torch.cuda.empty_cache()
        per_config = measure_per_config(ug, dev, peak)

    cpu = None
    if rank == 0 and G == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, size)
        cpu["single_thread"] = oracle_single_thread(cfg)

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": G,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "u8/u16 (integer)", "data": "synthetic (seeded; DESIGN.md section 4)",
            "config": {"workload": f"config 4: {size / 2**30:g} GiB mixed UTF-8 "
                                   "(60% ASCII/25% 2B/10% 3B/5% 4B), validate + UTF-8->UTF-16LE "
                                   "and back, sharded at character boundaries",
                       "bytes_utf8": N8, "units_utf16": N16,
                       "step": ("plan_utf8 (utf16_length_from_utf8 + range offsets) + "
                                "utf8_to_utf16le_planned + [allgather+combine] + plan_utf16le "
                                "(utf8_length_from_utf16le + range offsets) + "
                                "utf16le_to_utf8_planned + [allgather+combine]") if planned else
                               ("len16 + utf8_to_utf16le + [allgather+combine] + len8 + "
                                "utf16le_to_utf8 + [allgather+combine]"),
                       "path": args.path,
                       "parallelism": f"shard{G}", "l2": "inputs >= 1 GiB per rank > 126 MB L2; no flush",
                       "per_gpu_gbs": round(value / G, 2),
                       "gchar_per_s": round(gchar, 2), "gchar_per_s_per_gpu": round(gchar / G, 2),
                       "chars": NCH,
                       "forward_input_gbs": round(N8 / (fwd_ms * 1e-3) / 1e9 * 1, 2),
                       "gen_seconds": round(t_gen, 1)},
            "roofline": {"bound": "hbm", "achieved": round(D["achieved"], 1), "peak": peak,
                         "unit": "GB/s", "frac": round(D["frac"], 4),
                         "traffic": D["traffic"],
                         "traffic_source": D.get("traffic_source"),
                         "traffic_extrapolated": D.get("traffic_extrapolated"),
                         "kernel": f"{dom} ({D['op']}), the longest launch of the step",
                         "algorithmic_bytes_per_launch": alg_bytes,
                         "avg_launch_ms": round(D["ms"], 4), "peak_source": peak_src,
                         "issue": D["issue"],
                         "kernels": {k: {"op": d["op"], "avg_launch_ms": round(d["ms"], 4),
                                         "achieved": round(d["achieved"], 1),
                                         "frac": round(d["frac"], 4), "traffic": d["traffic"],
                                         "issue": d["issue"]}
                                     for k, d in kern.items()}},
            "per_op": per_op,
            "per_config": per_config,
            "clocks": clk,
            "gpu_launches": int(launches),
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        s = json.dumps(line)
        print(s, flush=True)
        if args.out:
            with open(args.out, "w") as f:
                f.write(s + "\n")
    if G > 1:
        dist.barrier()
        dist.destroy_process_group()


def measure_per_op(ug, t_all, off, n8, hb, ha, out16, u16, out8, dev, peak, reps=5):
    """Each hot-path op alone on this rank's shard (after the timed step; same buffers):
    mean CUDA-event time over `reps`, input GB/s, algorithmic HBM GB/s and its fraction of the
    measured copy peak.  Rows a1-a11 of SURVEY 8(a) individually."""
    import torch
    stream = torch.cuda.current_stream()
    t_in = t_all[off:off + n8]
    n16 = u16.numel()
    res = ug.result_buffer(dev, 1)
    lens = torch.zeros(1, dtype=torch.int64, device=dev)
    rec = ug.record_buffer(dev, 1)
    p8, p16 = ug.plan_buffer(dev), ug.plan_buffer(dev)
    ug.utf8_shard_plan_async(t_all, off, n8, hb, ha, lens, p8)
    ug.utf16le_shard_plan_async(u16, 0, n16, 0, 0, lens, p16)
    ops = {
        "utf8_validate": (lambda: ug.utf8_validate_async(t_in, res), n8, n8),
        "utf8_to_utf16le": (lambda: ug.utf8_to_utf16le_shard_async(
            t_all, off, n8, hb, ha, 0, out16, rec), n8, n8 + 2 * n16),
        "utf16_length_from_utf8": (lambda: ug.utf16_length_from_utf8_async(t_in, lens), n8, n8),
        "utf16le_validate": (lambda: ug.utf16le_validate_async(u16, res), 2 * n16, 2 * n16),
        "utf16le_to_utf8": (lambda: ug.utf16le_to_utf8_shard_async(
            u16, 0, n16, 0, 0, 0, out8, rec), 2 * n16, 2 * n16 + n8),
        "utf8_length_from_utf16le": (lambda: ug.utf8_length_from_utf16le_async(u16, lens),
                                     2 * n16, 2 * n16),
        # the two-pass form: the sizing passes with their plans, the planned transcoders
        "plan_utf8 (len16 + plan)": (lambda: ug.utf8_shard_plan_async(t_all, off, n8, hb, ha,
                                                                       lens, p8), n8, n8),
        "utf8_to_utf16le_planned": (lambda: ug.utf8_to_utf16le_shard_planned_async(
            t_all, off, n8, hb, ha, 0, p8, out16, rec), n8, n8 + 2 * n16),
        "plan_utf16le (len8 + plan)": (lambda: ug.utf16le_shard_plan_async(u16, 0, n16, 0, 0,
                                                                            lens, p16),
                                       2 * n16, 2 * n16),
        "utf16le_to_utf8_planned": (lambda: ug.utf16le_to_utf8_shard_planned_async(
            u16, 0, n16, 0, 0, 0, p16, out8, rec), 2 * n16, 2 * n16 + n8),
        # SURVEY 8(f) f4 (research comparison): the planned forward, keyed 12-byte decoder
        "utf8_to_utf16le_keyed (f4)": (lambda: ug.utf8_to_utf16le_keyed_planned_async(
            t_in, pk, out16, res), n8, n8 + 2 * n16),
    }
    pk = ug.plan_buffer(dev)
    ug.utf16_length_from_utf8_plan_async(t_in, lens, pk)
    out = {}
    for name, (fn, in_bytes, hbm_bytes) in ops.items():
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        out[name] = {"ms": round(ms, 4), "input_gbs": round(in_bytes / ms / 1e6, 1),
                     "hbm_gbs": round(hbm_bytes / ms / 1e6, 1),
                     "frac_of_peak": round(hbm_bytes / ms / 1e6 / peak, 4)}
    return out


def measure_per_config(ug, dev, peak, reps=50, reps_c0=2000):
    """Every hot-path op on BASELINE configs 0, 1, 2A, 2B and 3 at their BASELINE.json sizes
    (BASELINE.md section 2's targets): per op 3 warm-up calls, then
    `reps` async calls (2000 for config 0, which is L2-resident and launch-bound: reported, not a
    target), each bracketed by CUDA events on the stream; the minimum and mean call time, input
    GB/s, Gchar/s, algorithmic HBM GB/s and its fraction of the measured copy peak and of the
    nominal 8 TB/s (from the mean), and `spread_flag` when (mean - min) / min > 1 %.  Each
    config's other-encoding counterpart (its transcoded output) is produced by the library on
    the device first, so every op runs on that config's text."""
    import torch
    stream = torch.cuda.current_stream()
    res = ug.result_buffer(dev, 1)
    lens = torch.zeros(1, dtype=torch.int64, device=dev)
    out = {}
    for key in ("c0", "c1", "c2a", "c2b", "c3"):
        cfg = synth.CONFIGS[key]
        x = synth.generate(key)
        if cfg.encoding == "utf8":
            t8 = torch.from_numpy(x).to(dev)
            n16 = ug.utf16_length_from_utf8(t8)
            u16 = torch.empty(n16, dtype=torch.int16, device=dev)
            assert ug.utf8_to_utf16le(t8, u16).error == 0
        else:
            u16 = torch.from_numpy(x.view(np.int16)).to(dev)
            n8 = ug.utf8_length_from_utf16le(u16)
            t8 = torch.empty(n8, dtype=torch.uint8, device=dev)
            assert ug.utf16le_to_utf8(u16, t8).error == 0
        del x
        n8, n16 = t8.numel(), u16.numel()
        chars = int(((t8 & 0xC0) != 0x80).sum())
        o16 = torch.empty(n8, dtype=torch.int16, device=dev)
        o8 = torch.empty(n8 + 64, dtype=torch.uint8, device=dev)
        ops = {
            "utf8_validate": (lambda: ug.utf8_validate_async(t8, res), n8, n8),
            "utf8_to_utf16le": (lambda: ug.utf8_to_utf16le_async(t8, o16, res), n8, n8 + 2 * n16),
            "utf16_length_from_utf8": (lambda: ug.utf16_length_from_utf8_async(t8, lens), n8, n8),
            "utf16le_validate": (lambda: ug.utf16le_validate_async(u16, res), 2 * n16, 2 * n16),
            "utf16le_to_utf8": (lambda: ug.utf16le_to_utf8_async(u16, o8, res), 2 * n16,
                                2 * n16 + n8),
            "utf8_length_from_utf16le": (lambda: ug.utf8_length_from_utf16le_async(u16, lens),
                                         2 * n16, 2 * n16),
        }
        p8, p16 = ug.plan_buffer(dev), ug.plan_buffer(dev)
        ug.utf16_length_from_utf8_plan_async(t8, lens, p8)
        ug.utf8_length_from_utf16le_plan_async(u16, lens, p16)
        ops.update({
            "plan_utf8 (len16 + plan)": (lambda: ug.utf16_length_from_utf8_plan_async(
                t8, lens, p8), n8, n8),
            "utf8_to_utf16le_planned": (lambda: ug.utf8_to_utf16le_planned_async(
                t8, p8, o16, res), n8, n8 + 2 * n16),
            "plan_utf16le (len8 + plan)": (lambda: ug.utf8_length_from_utf16le_plan_async(
                u16, lens, p16), 2 * n16, 2 * n16),
            "utf16le_to_utf8_planned": (lambda: ug.utf16le_to_utf8_planned_async(
                u16, p16, o8, res), 2 * n16, 2 * n16 + n8),
            "utf8_to_utf16le_keyed (f4)": (lambda: ug.utf8_to_utf16le_keyed_planned_async(
                t8, p8, o16, res), n8, n8 + 2 * n16),
        })
        row = {"input": cfg.desc, "bytes_utf8": n8, "units_utf16": n16, "chars": chars}
        nrep = reps_c0 if key == "c0" else reps
        for name, (fn, in_bytes, hbm_bytes) in ops.items():
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(nrep + 1)]
            ev[0].record(stream)
            for r in range(nrep):
                fn()
                ev[r + 1].record(stream)
            torch.cuda.synchronize()
            t = [ev[r].elapsed_time(ev[r + 1]) for r in range(nrep)]
            ms, mn = sum(t) / nrep, min(t)
            row[name] = {"ms": round(ms, 4), "min_ms": round(mn, 4),
                         "input_gbs": round(in_bytes / ms / 1e6, 1),
                         "gchar_per_s": round(chars / ms / 1e6, 1),
                         "hbm_gbs": round(hbm_bytes / ms / 1e6, 1),
                         "frac_of_peak": round(hbm_bytes / ms / 1e6 / peak, 4),
                         "frac_of_8tbs": round(hbm_bytes / ms / 1e6 / 8000.0, 4),
                         "spread_flag": (ms - mn) / mn > 0.01}
        out[key] = row
        del t8, u16, o16, o8
        torch.cuda.empty_cache()
    return out


def run_e2e(args, ug, host_shard, n16, G, rank, dev, dist):
    """Same step through the public host-buffer API: H2D of the step's input from pinned host
    memory, the fused kernel, D2H of the result, both directions; wall clock, max over ranks."""
    import torch
    n8 = host_shard.size
    hin = torch.from_numpy(host_shard).pin_memory()
    h16 = torch.empty(n8, dtype=torch.int16).pin_memory()
    h8 = torch.empty(n8, dtype=torch.uint8).pin_memory()
    K = max(1, args.e2e_steps)
    ug.utf8_to_utf16le_host(hin[:1 << 20], h16)      # warm the staging buffers
    times = []
    for _ in range(K + 1):
        if G > 1:
            dist.barrier()
        t = time.perf_counter()
        r1 = ug.utf8_to_utf16le_host(hin, h16)
        r2 = ug.utf16le_to_utf8_host(h16[: r1.written], h8)
        times.append(time.perf_counter() - t)
        assert r1 == (0, n8, n16) and r2 == (0, n16, n8), (r1, r2)
    dt = min(times[1:]) if len(times) > 1 else times[0]
    tt = torch.tensor([dt, float(n8), float(n16)], dtype=torch.float64,
                      device=dev if args.dist_backend == "nccl" else "cpu")
    if G > 1:
        a = tt[:1].clone()
        dist.all_reduce(a, op=dist.ReduceOp.MAX)
        b = tt[1:].clone()
        dist.all_reduce(b, op=dist.ReduceOp.SUM)
        dt, N8, N16 = float(a[0]), int(b[0]), int(b[1])
    else:
        N8, N16 = n8, n16
    assert bytes(h8[:1 << 16].numpy()) == host_shard[:1 << 16].tobytes()
    return {"value": round((N8 + 2 * N16) / dt / 1e9, 3), "unit": UNIT,
            "h2d_bytes_per_step": N8 + 2 * N16, "d2h_bytes_per_step": 2 * N16 + N8,
            "steps": K, "api": "utf8_to_utf16le_host + utf16le_to_utf8_host (pinned)",
            "seconds_per_step": round(dt, 4)}


# ------------------------------------------------------------------------------ CPU legs
def oracle_step(oracle, chunk: np.ndarray):
    """The hot path on the CPU oracle, as it stands: sizing, forward, sizing, reverse."""
    n16 = oracle.utf16_length_from_utf8(chunk)
    r1, u = oracle.utf8_to_utf16le(chunk, out_cap=n16)
    n8 = oracle.utf8_length_from_utf16le(u)
    r2, back = oracle.utf16le_to_utf8(u, out_cap=n8)
    assert r1.error == 0 and r2.error == 0 and back.size == chunk.size
    return chunk.size + 2 * u.size


def oracle_single_thread(cfg, nbytes=64 << 20):
    """the oracle on ONE host core (the process pinned to it for
    the measurement), the same four-op step on one 64 MiB chunk of the workload."""
    import oracle
    oracle.build()
    data = np.frombuffer(synth.gen_chunk(cfg.mix, cfg.encoding, nbytes, cfg.seed, 0),
                         dtype=np.uint8)
    prev = os.sched_getaffinity(0) if hasattr(os, "sched_getaffinity") else None
    core = min(prev) if prev else None
    try:
        if core is not None:
            os.sched_setaffinity(0, {core})
        t = time.perf_counter()
        tot = oracle_step(oracle, data)
        dt = time.perf_counter() - t
    finally:
        if prev is not None:
            os.sched_setaffinity(0, prev)
    cpu = ""
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                cpu = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"value": round(tot / dt / 1e9, 4), "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"1 x {nbytes >> 20} MiB chunk of config {cfg.key}, pinned to core {core}; "
                      f"step = len16 + utf8->utf16le + len8 + utf16le->utf8",
            "seconds": round(dt, 2), "cpu_model": cpu}


def cpu_baseline(cfg, size, chunks=None):
    """The oracle on the host cores: independent 64 MiB generator chunks (each is whole,
    valid text, so the unmodified oracle runs on each), one per thread (ctypes releases the
    GIL).  Bounded sample: min(#cores, 16) chunks."""
    import oracle
    oracle.build()
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    nch = chunks or max(1, min(cores, 16, size // synth.CHUNK))
    data = [np.frombuffer(synth.gen_chunk(cfg.mix, cfg.encoding, min(synth.CHUNK, size),
                                          cfg.seed, c), dtype=np.uint8) for c in range(nch)]
    t = time.perf_counter()
    with ThreadPoolExecutor(nch) as ex:
        tot = sum(ex.map(lambda c: oracle_step(oracle, c), data))
    dt = time.perf_counter() - t
    return {"value": round(tot / dt / 1e9, 4), "unit": UNIT, "cores": nch, "kind": "oracle",
            "sample": f"{nch} x 64 MiB chunks of config {cfg.key} (first chunks), one per "
                      f"thread; step = len16 + utf8->utf16le + len8 + utf16le->utf8",
            "seconds": round(dt, 2), "host_cpus": cores}


def run_reference(args):
    """--impl reference: the oracle (no reference implementation exists for this paper) on
    the host cores, same metric/unit/config, each step a bounded sample."""
    G, rank, _ = dist_env()
    if rank != 0:
        return
    import oracle
    oracle.build()
    cfg = synth.CONFIGS[args.config]
    size = cfg.size if not args.size_mib else args.size_mib << 20
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    nch = max(1, min(cores, 8, size // synth.CHUNK))
    # exactly K timed and W warm-up steps; each step is a bounded sample (nch chunks, one per
    # thread) sized so the whole run stays near REF_BUDGET_S (a 64 MiB chunk takes ~1.2 s)
    K, W = max(1, args.steps), max(0, args.warmup)
    REF_BUDGET_S = 90.0
    frac = min(1.0, REF_BUDGET_S / ((K + W) * 1.3))
    clen = max(1 << 20, int(min(synth.CHUNK, size) * frac) >> 20 << 20)
    data = [np.frombuffer(synth.gen_chunk(cfg.mix, cfg.encoding, clen, cfg.seed, c),
                          dtype=np.uint8) for c in range(nch)]
    ex = ThreadPoolExecutor(nch)
    for _ in range(W):
        sum(ex.map(lambda c: oracle_step(oracle, c), data))
    t = time.perf_counter()
    tot = 0
    for _ in range(K):
        tot += sum(ex.map(lambda c: oracle_step(oracle, c), data))
    dt = (time.perf_counter() - t) / K
    v = (tot / K) / dt / 1e9
    line = {"impl": "reference", "metric": METRIC, "value": round(v, 4), "unit": UNIT,
            "n_gpus": G, "steps": K, "warmup": W,
            "ms_per_step": round(dt * 1e3, 2), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u8/u16 (integer)", "data": "synthetic",
            "config": {"workload": f"config 4 sample: {nch} x {clen >> 20} MiB of the {cfg.key} stream",
                       "parallelism": f"{nch} host threads"},
            "cpu_baseline": {"value": round(v, 4), "unit": UNIT, "cores": nch, "kind": "oracle",
                             "sample": f"{nch} x {clen >> 20} MiB chunks per step"},
            "e2e": {"value": round(v, 4), "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
