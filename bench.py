#!/usr/bin/env python
"""Throughput bench for the Hazedefy dehaze hot path on B200 (BASELINE.json metric).

Default workload (config C3): 300 synthetic 1920x1080 RGB u8 hazy frames per
GPU, video mode at native resolution (resize_to=None), reference defaults
(15x15 patch, top 0.1%, alpha 0.8, omega 0.5, t_min 0.05, gamma 1.2).
One step = one pass of the fused device pipeline over all frames of the rank
(inputs resident in HBM, 1.87 GB > L2, so no cross-step L2 reuse).
Weak scaling: each rank dehazes its own 300-frame shard of a longer clip; the
per-frame airlight trace is all-gathered over NCCL every step (N > 1).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl ours|reference]

Prints ONE JSON line (rank 0).  ``value`` = megapixels/s over all ranks
(device-resident), ``e2e`` = the same through the host API with pinned host
buffers (H2D + pipeline + D2H inside the timed region), ``roofline`` = the
dominant kernel (K6 recover) against measured HBM bandwidth, ``cpu_baseline``
= the CPU oracle port of the reference on a bounded sample.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "megapixels/sec (frames/s at 1080p/4K) at 1/2/4/8 B200; % HBM roofline"

CONFIG_PARAMS = {
    "c1": dict(resize_to=None),
    "c3": dict(resize_to=None),
    "c4": dict(resize_to=None, white_balance=True),
    "c2": dict(mode="image", resize_to=None, guided_radius=30, guided_eps=1e-3),
    "c5": dict(mode="image", resize_to=None, patch_radius=15, guided_radius=60, guided_eps=1e-3),
    # the reference's default DehazeParams() (resize_to=(640, 480)) on the C3 frames (SURVEY §8(d),
    # "secondary row"; throughput counted in input megapixels)
    "c3d": dict(),
}


def engine_for_sizes(params, H, W):
    from paper_2512_16609_b200.engine import FrameEngine

    return FrameEngine.working_size(params, H, W)


def _size_note(params):
    if params.resize_to is None:
        return "native resolution"
    return f"resized to {params.resize_to[0]}x{params.resize_to[1]} (reference default; MP/s counts input pixels)"


def _base(cfg):
    """Synthetic frame config behind a bench config ("c3d" runs on the C3 frames)."""
    return cfg[:2]
# algorithmic HBM bytes per pixel: dark 4 + select 1 + recover 6 (+3 balance);
# image mode + balance 29 (dark 4 + select 1 + guided 7 (read I 3, write t~ fp32 4) + recover 6
# + t~ read 4 + balance 3 + 4).  The exact two-pass guided filter's own design moves more
# (pass 1 writes the fixed-point a, b 16 B/px, pass 2 reads them for the entering and the
# leaving row 32, t~ is fp64 8 written + 8 read, apply reads I again 3): DESIGN_BYTES,
# reported beside it (4 + 1 + (3 + 16) + (32 + 3 + 8) + (8 + 3 + 3) = 81 B/px).
ALG_BYTES = {"c1": 11, "c3": 11, "c4": 14, "c2": 29, "c5": 29,
             # resize path per INPUT pixel (1080p -> 640x480, 0.148 output px per input px): dark pass
             # reads I 3 + writes dark 8*0.148, select reads dark 8*0.148, recover reads I 3 + writes 3*0.148
             "c3d": round(6 + 19 * (640 * 480) / (1920 * 1080), 2)}
DESIGN_BYTES = {"c2": 81, "c5": 81}
# the guided stage (guided filter + recovery [+ balance]) at §8(d) bytes: 29 - dark 4 - select 1
GUIDED_BYTES = {False: 13, True: 24}


def _guided_chunk(n, H, W, params):
    """Frames per guided-filter chunk (csrc/guided_fused.cu x_chunk, the default two-pass form)."""
    per = (24.0 if params.balance_enabled() else 16.0) * H * W
    cap = int(max(1.0, min(float(n), 12.0e9 / per)))
    chunks = (n + cap - 1) // cap
    return (n + chunks - 1) // chunks


def _ncu_traffic_per_px():
    """DRAM bytes per pixel per kernel from the committed ncu capture (profiles/ncu_traffic.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            return {k: float(v["dram_bytes_per_px"]) for k, v in json.load(fh)["kernels"].items()}
    except Exception:
        return {}


def _ncu_guided_traffic_per_px(balance):
    """DRAM bytes per pixel of the image-mode guided stage (its kernels summed) from the committed
    ncu launch list of the C5 bench command (profiles/ncu_traffic_c5.json); None if absent."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic_c5.json")) as fh:
            ks = json.load(fh)["kernels"]
        names = ["k_gx_ab", "k_gx_out"] + (["k_gw_sums", "k_gf_thresholds", "k_gf_apply2"] if balance else [])
        return sum(float(ks[k]["dram_bytes_per_px"]) for k in names if k in ks)
    except Exception:
        return None


def _calibration(cfg):
    """Real reference vs the oracle port on identical frames (tools/calibrate_cpu_baseline.py, run
    where /root/reference exists; one thread each): how much slower the reference itself is."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02_cpu_baseline_calibration.json")) as fh:
            d = json.load(fh).get(_base(cfg))
        return {"reference_time_over_port": d["port_over_reference"], "identical_outputs": d["identical_outputs"],
                "source": "profiles/r02_cpu_baseline_calibration.json (survey container, 1 thread, "
                          f"{d['frames']} {_base(cfg)} frames)"}
    except Exception:
        return None


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        sm.sort()
        med = sm[len(sm) // 2] if sm else None
        return {"sm_mhz": med, "sm_max_mhz": smax, "reasons": sorted(reasons), "samples": len(sm)}


def cpu_baseline(frames_np, params, workers, budget_s=20.0):
    """Time the CPU oracle (numpy port of the reference) on a bounded sample, all host cores."""
    from oracle import dehaze_oracle

    npx = frames_np.shape[1] * frames_np.shape[2]
    done = 0
    t0 = time.perf_counter()
    while True:
        dehaze_oracle.process_stream(list(frames_np), params, workers=workers)
        done += frames_np.shape[0]
        el = time.perf_counter() - t0
        if el >= budget_s * 0.5:
            break
    return done * npx / el / 1e6, done, el


def run_reference(args):
    """--impl reference: the CPU oracle port of the reference path on this box's host cores."""
    import numpy as np
    import torch

    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import dehaze_oracle  # noqa: F401
    from paper_2512_16609_b200.pipeline import DehazeParams
    from paper_2512_16609_b200.synthetic import CONFIGS, make_frames

    cfg = args.config
    spec = CONFIGS[_base(cfg)]
    params = DehazeParams(**CONFIG_PARAMS[cfg])
    workers = os.cpu_count() or 1
    sample = max(1, min(spec["frames"], workers))
    frames = make_frames(_base(cfg), frames=sample).numpy()
    npx = frames.shape[1] * frames.shape[2]
    from oracle.dehaze_oracle import process_stream

    for _ in range(args.warmup and 1):
        process_stream(list(frames[:1]), params, workers=1)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        process_stream(list(frames), params, workers=workers)
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    value = sample * npx * args.steps / tot / 1e6
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": round(value, 3),
        "unit": "MP/s",
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(1000 * tot / args.steps, 3),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded BASELINE generator)",
        "config": {"workload": f"{cfg}: {sample} of {spec['frames']} frames {spec['width']}x{spec['height']} "
                               f"per step, {params.mode} mode, " + _size_note(params),
                   "frames_per_step": sample},
        "cpu_baseline": {"value": round(value, 3), "unit": "MP/s", "cores": workers, "kind": "port",
                         "sample": f"{sample} frames per step, oracle/dehaze_oracle.py process_stream "
                                   f"workers={workers}", "calibration": _calibration(cfg)},
        "e2e": {"value": round(value, 3), "unit": "MP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _count_launches(fn, stream):
    """Kernels of this package launched by one call of ``fn`` (CUDA-graph replays included),
    from a torch.profiler (CUPTI) trace; (None, None) if the profiler is unavailable."""
    import torch

    try:
        from torch.profiler import ProfilerActivity, profile

        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            fn()
            torch.cuda.synchronize()
        names = {}
        for ev in prof.events():
            nm = ev.name or ""
            if "dhz::" in nm or nm.startswith("_ZN3dhz") or "k_ema" in nm:
                import re

                m = re.search(r"(k_\w+)", nm)
                key = m.group(1) if m else nm[:60]
                names[key] = names.get(key, 0) + 1
        total = sum(names.values())
        return (total if total else None), names
    except Exception:
        return None, None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c3", choices=sorted(CONFIG_PARAMS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="eager launches instead of a CUDA-graph replay per step")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # DHZ_BENCH_SHARDED=1 takes the N>1 code path (process group, dehaze_sharded steps) in a
    # world of one, so the path can be exercised on a one-GPU lease under torchrun
    sharded = world > 1 or os.environ.get("DHZ_BENCH_SHARDED") == "1"
    if sharded:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29531")
        dist.init_process_group("nccl", device_id=dev, rank=rank, world_size=world)

    from paper_2512_16609_b200.engine import engine_for
    from paper_2512_16609_b200.pipeline import DehazeParams, dehaze_host_batch
    from paper_2512_16609_b200.synthetic import CONFIGS, Scene, make_frames

    cfg = args.config
    spec = CONFIGS[_base(cfg)]
    params = DehazeParams(**CONFIG_PARAMS[cfg])
    n, H, W = spec["frames"], spec["height"], spec["width"]
    npx = H * W
    OH, OW = engine_for_sizes(params, H, W)

    # ---- inputs: this rank's shard, generated on the device -------------------
    frames = torch.empty((n, H, W, 3), dtype=torch.uint8, device=dev)
    base = _base(cfg)
    if base in ("c3", "c4", "c1", "c2"):
        scene = Scene(W, H, 1000 * int(base[1:]), dev)
        for f in range(n):
            g = rank * n + f
            beta = 0.65 - 0.15 * math.cos(2 * math.pi * g / 300.0) if base in ("c3", "c4") else 0.6
            frames[f] = scene.hazy_u8(g, 1000 * int(base[1:]) + g, beta, spec["airlight"])
    else:
        make_frames(base, frames=n, device=dev, out=frames)
    torch.cuda.synchronize()

    from paper_2512_16609_b200.pipeline import _native_ok, dehaze_batch

    native = _native_ok(params, H, W)
    eng = engine_for(dev)
    out = torch.empty((n, OH, OW, 3), dtype=torch.uint8, device=dev)
    air = torch.empty((n, 3), dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)
    n_ev = 5
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(n_ev)] for _ in range(args.steps)]

    graph = None
    if native and not args.no_graph and not sharded:
        # the batch pipeline captured once as a CUDA graph and replayed per step
        # (same kernels on the same buffers; removes the per-launch gaps)
        from paper_2512_16609_b200.engine import GraphedPipeline
        # timed graph: no stage-event nodes (each costs ~4 us of the step: 22 us of
        # C3's 1.55 ms, 18 us of C1's 0.07 ms); a second graph of the same kernels on
        # the same buffers carries the stage events and is replayed right after the
        # timed region for the per-stage (and K6 roofline) times
        graph_ev = [torch.cuda.Event(enable_timing=True) for _ in range(n_ev)]
        graph = GraphedPipeline(frames, params, out=out, airlight=air, streams=1)
        graph_st = GraphedPipeline(frames, params, out=out, airlight=air, streams=1, events=graph_ev)

    shard_pipe = None
    if sharded and native and not args.no_graph:
        # the product's multi-GPU path with its two halves captured as CUDA graphs
        from paper_2512_16609_b200.distributed import ShardedPipeline

        shard_pipe = ShardedPipeline(frames, params, n * world)

    def step(ev=None):
        nonlocal out, air
        if sharded:
            # the product's multi-GPU path: airlight half on this rank's shard, NCCL
            # all-gather of the trace (24 B/frame), recovery half (distributed.dehaze_sharded
            # / ShardedPipeline)
            if shard_pipe is not None:
                out, _trace = shard_pipe.step()
            else:
                from paper_2512_16609_b200.distributed import dehaze_sharded

                out, _trace = dehaze_sharded(frames, params, n * world)
            if ev is not None:
                for e in ev:
                    e.record(stream)
            return
        if native and graph is not None and ev is None:
            graph.replay()
        elif native:
            eng.run(frames, params, out=out, airlight=air, stream=stream, events=ev)
        else:  # image mode: float64 device path, frame by frame
            out, air = dehaze_batch(frames, params)
            if ev is not None:
                for e in ev:
                    e.record(stream)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    if sharded:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    # L2 (126 MB): inputs + outputs of a step smaller than 2x L2 could be served from it
    # across steps, so such configs write a 512 MB buffer between timed steps
    in_out_bytes = n * 3 * (npx + OH * OW)
    flush = torch.zeros(128 << 20, dtype=torch.int32, device=dev) if in_out_bytes < (256 << 20) else None
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if sharded:
        dist.barrier()
    if flush is None:  # inputs larger than L2: back-to-back steps, one event pair
        t_start.record(stream)
        for k in range(args.steps):
            step(None if graph is not None else evs[k])
        t_end.record(stream)
        torch.cuda.synchronize()
        ms = t_start.elapsed_time(t_end)
    else:  # inputs fit in L2: flush it between steps, outside each step's event pair
        pairs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                 for _ in range(args.steps)]
        for k in range(args.steps):
            flush.add_(1)
            pairs[k][0].record(stream)
            step(None if graph is not None else evs[k])
            pairs[k][1].record(stream)
        torch.cuda.synchronize()
        ms = sum(a.elapsed_time(b) for a, b in pairs)
    clk = clocks.stop()
    if sharded:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    total_px = n * npx * world
    value = total_px / (ms_step / 1000.0) / 1e6

    # per-stage device times (event i -> i+1): eager steps average over the timed
    # steps; graph replays re-record the captured stage events, which then hold the
    # last timed step
    stage_ms = [0.0] * (n_ev - 1)
    if graph is not None:
        for _ in range(args.steps):
            if flush is not None:
                flush.add_(1)
            graph_st.replay()
            torch.cuda.synchronize()
            for i in range(n_ev - 1):
                stage_ms[i] += graph_ev[i].elapsed_time(graph_ev[i + 1]) / args.steps
    else:
        if sharded and native:
            # sharded steps carry no stage events (two halves around a collective): the stage
            # times come from eager runs of the same kernels over this rank's shard, after
            # the timed region
            for k in range(args.steps):
                if flush is not None:
                    flush.add_(1)
                eng.run(frames, params, out=out, airlight=air, stream=stream, events=evs[k])
            torch.cuda.synchronize()
        for k in range(args.steps):
            for i in range(n_ev - 1):
                stage_ms[i] += evs[k][i].elapsed_time(evs[k][i + 1]) / args.steps
    if sharded:  # the roofline's launch time is the slowest rank's
        t = torch.tensor(stage_ms, device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        stage_ms = [float(v) for v in t.tolist()]
    peak, peak_kind = _peaks()
    pipe_bytes = ALG_BYTES[cfg] * n * npx
    pipe_gbs = pipe_bytes / (ms_step / 1000.0) / 1e9
    traffic_px = _ncu_traffic_per_px()
    if native and (OH, OW) != (H, W):
        rec_bytes = n * (3 * npx + 3 * OH * OW)   # R3: read I (3 B/input px), write O (3 B/output px)
        rec_gbs = rec_bytes / (stage_ms[3] / 1000.0) / 1e9
        roof = {"bound": "hbm", "kernel": "k_rs_recover (R3, resize + recovery, fp64)", "achieved": round(rec_gbs, 1),
                "peak": peak, "unit": "GB/s", "frac": round(rec_gbs / peak, 4), "traffic": None,
                "peak_kind": peak_kind, "alg_bytes_per_launch": rec_bytes, "launch_ms": round(stage_ms[3], 4)}
        launches = 3 + (2 if params.balance_enabled() else 0)
    elif native and params.mode == "video":
        rec_bytes = 6 * n * npx          # K6: read I (3 B/px), write O (3 B/px)
        rec_gbs = rec_bytes / (stage_ms[3] / 1000.0) / 1e9
        t_px = traffic_px.get("k_recover_lut_diag")
        roof = {"bound": "hbm", "kernel": "k_recover_lut_diag (K6, LUT recovery)", "achieved": round(rec_gbs, 1),
                "peak": peak, "unit": "GB/s", "frac": round(rec_gbs / peak, 4),
                "traffic": None if t_px is None else int(t_px * n * npx), "peak_kind": peak_kind,
                "alg_bytes_per_launch": rec_bytes, "launch_ms": round(stage_ms[3], 4),
                "traffic_source": "profiles/ncu_traffic.json (ncu dram__bytes_read+write per px)"}
        # K1, K2 level hist, K3 threshold, 2 fallback kernels (exit at once on the fast
        # path), K3c compact, K4 airlight, K5 LUT (balance: g table, sums, LUT), K6
        launches = 9 + (2 if params.balance_enabled() else 0)
    elif native:
        gb = GUIDED_BYTES[params.balance_enabled()] * n * npx
        g_gbs = gb / (stage_ms[2] / 1000.0) / 1e9
        roof = {"bound": "hbm", "kernel": "guided stage at SURVEY §8(d) bytes (%d B/px): k_gx_ab + k_gx_out "
                "(+ k_gf_thresholds + k_gf_apply2)" % GUIDED_BYTES[params.balance_enabled()],
                "achieved": round(g_gbs, 1), "peak": peak, "unit": "GB/s", "frac": round(g_gbs / peak, 4),
                "traffic": None, "peak_kind": peak_kind, "alg_bytes_per_launch": gb,
                "launch_ms": round(stage_ms[2], 4)}
        tpx = _ncu_guided_traffic_per_px(params.balance_enabled()) if _base(cfg) == "c5" else None
        if tpx is not None:  # measured on C5 frames (8K, r = 60); other geometries differ, so C2 stays null
            roof["traffic"] = int(round(tpx * n * npx))
            roof["traffic_source"] = "profiles/ncu_traffic_c5.json (ncu dram__bytes_read+write per px, stage kernels summed)"
        # K1 + the 6 select kernels + pass1 + pass2 (+ sums, thresholds, apply) per <=12 GB chunk of frames
        launches = 7 + (5 if params.balance_enabled() else 2) * math.ceil(n / _guided_chunk(n, H, W, params))
    else:
        roof = {"bound": "hbm", "kernel": "float64 image-mode pipeline (whole step)", "achieved": round(pipe_gbs, 1),
                "peak": peak, "unit": "GB/s", "frac": round(pipe_gbs / peak, 4), "traffic": None,
                "peak_kind": peak_kind, "alg_bytes_per_launch": pipe_bytes, "launch_ms": round(ms_step, 4)}
        launches = 24 * n

    formula_launches = launches
    launches, launch_names = _count_launches(lambda: step(None), stream)
    launch_source = "counted: kernels of libdehaze_b200.so in one step under torch.profiler (CUPTI)"
    if launches is None:
        launches, launch_source = formula_launches, "formula (profiler unavailable)"

    # ---- e2e: host API with pinned buffers ----------------------------------
    e2e = None
    if args.e2e_steps > 0:
        host_in = torch.empty((n, H, W, 3), dtype=torch.uint8, pin_memory=True)
        host_in.copy_(frames)
        host_out = torch.empty((n, OH, OW, 3), dtype=torch.uint8, pin_memory=True)
        host_air = torch.empty((n, 3), dtype=torch.float64, pin_memory=True)
        dehaze_host_batch(host_in, params, out=host_out, airlight=host_air)   # warm-up
        torch.cuda.synchronize()
        if sharded:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            dehaze_host_batch(host_in, params, out=host_out, airlight=host_air)
        torch.cuda.synchronize()
        el = (time.perf_counter() - t0) / args.e2e_steps
        if sharded:
            t = torch.tensor([el], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            el = float(t.item())
        e2e = {"value": round(total_px / el / 1e6, 3), "unit": "MP/s",
               "h2d_bytes_per_step": int(host_in.numel()), "d2h_bytes_per_step": int(host_out.numel() + 24 * n),
               "ms_per_step": round(1000 * el, 3)}
        ok = torch.equal(host_out, out.cpu())
        e2e["matches_device_path"] = bool(ok)
        # the reference's own entry point: process_stream over a list of numpy frames
        # (pinned staging filled by the copy threads, fresh output arrays to the sink)
        from paper_2512_16609_b200.pipeline import process_stream

        frames_np = list(host_in.numpy())
        got = []
        process_stream(frames_np[: min(n, 8)], params, sink=got.append)   # warm-up
        del got
        sk = 0

        def sink(o):
            nonlocal sk
            sk += 1

        process_stream(frames_np, params, sink=sink)   # warm-up at full length (pinned output buffers cached)
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            st_ = process_stream(frames_np, params, sink=sink)
        el_s = (time.perf_counter() - t0) / args.e2e_steps
        if sharded:
            t = torch.tensor([el_s], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            el_s = float(t.item())
        e2e["process_stream"] = {"value": round(total_px / el_s / 1e6, 3), "unit": "MP/s",
                                 "ms_per_step": round(1000 * el_s, 3),
                                 "api": "process_stream(list of numpy frames, params, sink) (reference API)",
                                 "frames_emitted": st_.frame_count}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        workers = os.cpu_count() or 1
        sample = min(n, workers)
        v, done, el = cpu_baseline(frames[:sample].cpu().numpy(), params, workers)
        cpu = {"value": round(v, 3), "unit": "MP/s", "cores": workers, "kind": "port",
               "sample": f"{done} frames of the {cfg} workload ({W}x{H}) through oracle/dehaze_oracle.py "
                         f"process_stream(workers={workers}) in {el:.1f} s", "calibration": _calibration(cfg)}

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": round(value, 3),
            "unit": "MP/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": max(3, args.warmup),
            "ms_per_step": round(ms_step, 4),
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": ("f64 (resized image)" if (OH, OW) != (H, W) else
                      "u8" if params.mode == "video" else "u8 in/out, f64 guided filter") if native else "f64",
            "data": "synthetic (seeded BASELINE generator, generated on device)",
            "config": {"workload": f"{cfg}: {n} frames {W}x{H} per GPU, {params.mode} mode, " + _size_note(params)
                                   + (", gray-world balance" if params.balance_enabled() else ""),
                       "frames_per_gpu": n, "fps": round(n * world / (ms_step / 1000.0), 1),
                       "step": ("one CUDA-graph replay of the batch pipeline (no instrumentation in the "
                                "timed graph; stage times from the same pipeline captured with stage-event "
                                "nodes, replayed --steps times after the timed region)"
                                if graph is not None else
                                "airlight half (CUDA graph), NCCL all-gather of the airlight trace (eager), "
                                "recovery half (CUDA graph) (distributed.ShardedPipeline); stage times from eager runs of the same kernels "
                                "after the timed region, max over ranks" if sharded else
                                "eager launches of the batch pipeline"),
                       "l2": (f"inputs + outputs {in_out_bytes / 1e9:.2f} GB/step > 2x the 126 MB L2 "
                              "(no flush needed)" if flush is None else
                              f"inputs + outputs {in_out_bytes / 1e6:.1f} MB/step fit in L2: a 512 MB buffer "
                              "is written between timed steps (outside each step's event pair)"),
                       "params": {k: getattr(params, k) for k in ("patch_radius", "top_fraction", "alpha",
                                                                  "omega", "t_min", "gamma")}},
            "roofline": roof,
            "pipeline_roofline": {"alg_bytes_per_px": ALG_BYTES[cfg], "achieved": round(pipe_gbs, 1),
                                  **({"design_bytes_per_px": DESIGN_BYTES[cfg],
                                      "design_frac": round(DESIGN_BYTES[cfg] * n * npx / (ms_step / 1000.0) / 1e9
                                                           / peak, 4)} if cfg in DESIGN_BYTES else {}),
                                  "frac": round(pipe_gbs / peak, 4),
                                  "stage_ms": {"dark(K1)": round(stage_ms[0], 4),
                                               "select+airlight(K2-K3)": round(stage_ms[1], 4),
                                               **({"guided+recover": round(stage_ms[2], 4)}
                                                  if params.mode == "image" else
                                                  {"lut(K5)": round(stage_ms[2], 4),
                                                   "recover(K6)": round(stage_ms[3], 4)})}},
            "gpu_launches": launches * args.steps,
            "gpu_launches_source": launch_source,
            "gpu_launches_per_step": launch_names,
            "clocks": clk,
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if sharded:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
