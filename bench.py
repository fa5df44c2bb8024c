"""Benchmark: range-image segmentation throughput on B200 (BASELINE.json metric).

Workload (default): BASELINE config 1 — 256 independent 64x2048 float32 frames
(seeds 0-255 per rank), reference default parameters (ground removal on,
d_max 0.8 m, theta 10 deg, min_cluster_points 100, skip count S = 0, i.e. no
Map Connections).  One step = one fused kernel launch over the whole batch.

Prints ONE JSON line (rank 0).  ``value`` = frames/s over all ranks with the
inputs resident in HBM; ``e2e`` = the same metric through the host-buffer C
ABI (``rs_segment_batch_host``: pinned host ranges in, labels / counts / sizes
back to the host, copies inside the timed region); ``roofline`` = the kernel's
algorithmic bytes (16.5 B/cell) / its event-timed duration
against the measured HBM copy bandwidth; ``cpu_baseline`` = the CPU oracle
port of the reference path on this host's cores.

``--impl reference`` times the CPU oracle (the reference algorithm restated
in C, oracle/) with all host threads on the same workload and metric.

Multi-GPU (torchrun): each rank segments its own 256 frames (weak scaling,
no collective on the data path — frames are independent); the step time is
the max over ranks.
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
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

ALGO_BYTES_PER_CELL = 16.5          # 4 in + 4 out + 0.5 edge bits + 8 label scratch
MC_BYTES_PER_OFFSET = 0.25
COMPULSORY_BYTES_PER_CELL = 8.0


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=100)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--config", type=int, default=1, help="BASELINE config id (0-4)")
    p.add_argument("--skip", type=int, default=0, help="skip count S (0 = reference default)")
    p.add_argument("--core", action="store_true", help="ground off, min_cluster_points 1")
    p.add_argument("--rows-per-cta", type=int, default=0)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=10.0)
    p.add_argument("--no-cloud", action="store_true", help="skip the point-cloud path measurement")
    p.add_argument("--no-per-config", action="store_true", help="skip the per-config block")
    p.add_argument("--no-check", action="store_true", help="skip the parity checks against the oracle")
    p.add_argument("--no-frame-api", action="store_true", help="skip the per-frame API latency")
    return p.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def pipeline_config(args):
    import paper_2003_00575_b200 as rs
    if args.core:
        return rs.PipelineConfig(mc_pattern=rs.skip_pattern(args.skip), ground_removal=False,
                                 min_cluster_points=1)
    return rs.PipelineConfig(mc_pattern=rs.skip_pattern(args.skip))


def workload_config(args, spec, batch, world):
    return {
        "workload": f"BASELINE config {args.config}: {spec.name}",
        "frames_per_gpu": batch, "H": spec.H, "W": spec.W,
        "cells_per_gpu": batch * spec.H * spec.W,
        "params": ("core: ground off, min_cluster_points 1" if args.core else
                   "reference defaults: ground on, d_max 0.8, theta 10, min_cluster_points 100")
                  + f", skip S={args.skip}",
        "l2": "flushed between timed steps (512 MiB write); inputs 134 MB > L2 as well",
        "parallelism": f"replicas x{world} (independent frames, no collective)",
    }


def measured_peak():
    f = ROOT / "MEASURED_PEAKS.json"
    if f.exists():
        try:
            return float(json.loads(f.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
        except Exception:
            pass
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region.

    NVML (pynvml) polled from a thread every few milliseconds; falls back to
    ``nvidia-smi -lms`` (B200_PROFILING.md clocks line) when NVML is missing.
    """

    REASONS = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40),
               ("sw_thermal_slowdown", 0x20), ("sw_power_cap", 0x4))

    def __init__(self, index, period_s=0.005):
        self.index = index
        self.period = period_s
        self.samples = []
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        self._proc = None

    def _nvml_loop(self, pynvml, h):
        while not self._stop.is_set():
            try:
                sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append((sm, rs))
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            self._t = threading.Thread(target=self._nvml_loop, args=(pynvml, h), daemon=True)
            self._t.start()
        except Exception:
            try:
                self._proc = subprocess.Popen(
                    ["nvidia-smi", "-i", str(self.index),
                     "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                     "--format=csv,noheader,nounits", "-lms", "50"],
                    stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
                self._t = threading.Thread(target=self._smi_loop, daemon=True)
                self._t.start()
            except Exception:
                self._proc = None
        return self

    def _smi_loop(self):
        for line in self._proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            try:
                self.samples.append((float(parts[0]), int(parts[2], 16)))
                self.max_mhz = float(parts[1])
            except (ValueError, IndexError):
                continue

    def __exit__(self, *exc):
        self._stop.set()
        if self._proc is not None:
            self._proc.terminate()
        if self._t is not None:
            self._t.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        reasons = sorted({n for _, r in self.samples for n, bit in self.REASONS if r & bit})
        return {"sm_mhz": statistics.median(s for s, _ in self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.samples)}


def cpu_sample(frames_np, packed, seconds, nthreads=1):
    """Time the oracle port on whole frames until ~`seconds` of CPU work."""
    from oracle import oracle
    B = frames_np.shape[0]
    done, t0 = 0, time.perf_counter()
    chunk = max(1, nthreads)
    i = 0
    while True:
        sl = frames_np[i:i + chunk]
        oracle.segment_batch(sl, packed, nthreads=nthreads)
        done += sl.shape[0]
        i = (i + chunk) % B
        el = time.perf_counter() - t0
        if el >= seconds:
            return done, el


def cloud_bench(args, pipe, frames, spec, flush):
    """Point-cloud path (Pipeline.segment_cloud on B clouds):
    the config's frames back-projected to float64 points (one point per valid
    cell, cell-centre azimuth), resident in HBM; per step rs_project ->
    rs_segment_batch -> rs_labels_to_points, device-timed.  CPU: the oracle's
    project + segment + labels_to_points on two clouds, one thread."""
    import numpy as np
    import torch
    from paper_2003_00575_b200 import cloud
    dev = frames.device
    model = pipe.model
    r = frames.double()
    el = torch.as_tensor(np.asarray(model.channel_angles), dtype=torch.float64, device=dev)[:, None]
    az = (torch.arange(model.width, dtype=torch.float64, device=dev) + 0.5) * model.azimuth_step
    keep = r > 0
    xyz = torch.stack([r * torch.cos(el) * torch.cos(az), r * torch.cos(el) * torch.sin(az),
                       r * torch.sin(el).expand_as(r)], -1)
    pts = xyz[keep].contiguous()
    off = torch.zeros(frames.shape[0] + 1, dtype=torch.int64, device=dev)
    off[1:] = torch.cumsum(keep.flatten(1).sum(1), 0)
    n = int(off[-1].item())

    def step():
        ranges, pidx, _ = cloud.project_batch(pts, off, model)
        res = pipe.segment_batch(ranges)
        return cloud.labels_to_points_batch(res.labels, pidx, off)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    steps = max(5, args.steps // 10)
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(steps)]
    for e in ev:
        flush.zero_()
        e[0].record()
        ranges, pidx, _ = cloud.project_batch(pts, off, model)
        e[1].record()
        res = pipe.segment_batch(ranges)
        e[2].record()
        cloud.labels_to_points_batch(res.labels, pidx, off)
        e[3].record()
    torch.cuda.synchronize()
    tot = sum(e[0].elapsed_time(e[3]) for e in ev) / steps
    proj = sum(e[0].elapsed_time(e[1]) for e in ev) / steps
    seg = sum(e[1].elapsed_time(e[2]) for e in ev) / steps
    back = sum(e[2].elapsed_time(e[3]) for e in ev) / steps
    B = frames.shape[0]
    out = {"value": B / (tot * 1e-3), "unit": "clouds/s", "points_per_s": n / (tot * 1e-3),
           "points_per_cloud": n / B, "ms_per_step": tot, "steps": steps,
           "stages_ms": {"project": proj, "segment": seg, "labels_to_points": back},
           "path": "cloud.project_batch -> Pipeline.segment_batch -> cloud.labels_to_points_batch "
                   "(rs_project, rs_segment_batch, rs_labels_to_points), float64 points in HBM"}
    if not args.no_cpu_baseline:
        from oracle import oracle
        offs = off.cpu().numpy()
        host = pts[: int(offs[2])].cpu().numpy()
        t0 = time.perf_counter()
        for b in range(2):
            c = host[offs[b]:offs[b + 1]]
            wr, wp, _, _ = oracle.project(c, model)
            wl, _ = oracle.segment_frame(wr, pipe.packed)
            oracle.labels_to_points(wl, wp, len(c))
        el_s = time.perf_counter() - t0
        out["cpu_baseline"] = {"value": 2 / el_s, "unit": "clouds/s", "cores": 1, "kind": "port",
                               "sample": "2 clouds, oracle project + segment_frame + labels_to_points"}
    return out


def ref_pipe_args(args, spec):
    """Arguments of baseline/ref_bench.make_pipeline for this workload."""
    import paper_2003_00575_b200 as rs
    cfg = pipeline_config(args)
    return dict(H=spec.H, W=spec.W, top_deg=spec.top_deg, bottom_deg=spec.bottom_deg, mount=spec.mount,
                offsets=tuple(cfg.mc_pattern.offsets), ground=cfg.ground_removal,
                min_points=cfg.min_cluster_points)


def run_reference(args):
    """CPU arm: the UNMODIFIED reference (baseline/_ref, pure Python + numba)
    through its public Pipeline API, one process per host core; falls back to
    the C port of the reference algorithm (oracle/) if it is not installed."""
    rank, _, world = dist_env()
    if rank != 0:
        return
    from baseline import ref_bench
    from paper_2003_00575_b200 import synthetic
    spec = synthetic.CONFIGS[args.config]
    rangeseg, why = ref_bench.load()
    if rangeseg is None:
        return run_reference_port(args, why)
    # a bounded sample of the workload: its first frames (seeds 0..n-1),
    # generated on the host (no CUDA in this process: the workers fork)
    n = min(spec.batch, 32)
    frames = synthetic.make_batch(args.config, n, device="cpu").numpy()
    pa = ref_pipe_args(args, spec)
    one = ref_bench.single_core(frames[:16], pa, min_seconds=3.0)
    nproc = os.cpu_count() or 1
    per_proc = max(1, int(round(0.25 * one["frames_per_s"])))   # ~0.25 s of work per process and step
    pool = ref_bench.AllCores(frames, pa, nproc)
    for _ in range(args.warmup):
        pool.step(per_proc)
    done, tot = 0, 0.0
    for _ in range(args.steps):
        d, el = pool.step(per_proc)
        done += d
        tot += el
    pool.close()
    fps = done / tot
    cells = spec.H * spec.W
    line = {
        "impl": "reference", "metric": "frames/s", "value": fps, "unit": "frames/s",
        "points_per_s": fps * cells, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": tot / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded BASELINE generator)",
        "config": workload_config(args, spec, spec.batch, 1),
        "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": nproc, "kind": "reference",
                         "sample": f"{per_proc} frames per process and step cycling over the workload's first "
                                   f"{n} frames; {nproc} processes (one per core, pinned), each with its own "
                                   "rangeseg.Pipeline from baseline/_ref (unmodified reference, "
                                   "segment_range_image)",
                         "cpu_model": ref_bench.cpu_model()},
        "single_core": dict(one, semantics="rangeseg.bench_run: 1 pinned core, GC off, warm-up 3, "
                                           "per-frame TimingRecord.total"),
        "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_reference_port(args, why):
    """Fallback reference arm: the C port of the reference algorithm (oracle/)."""
    rank, _, world = dist_env()
    import torch
    import paper_2003_00575_b200 as rs
    from oracle import oracle
    from paper_2003_00575_b200 import synthetic
    spec = synthetic.CONFIGS[args.config]
    frames = synthetic.make_batch(args.config, device="cuda" if torch.cuda.is_available() else "cpu")
    frames_np = frames.cpu().numpy()
    packed = rs.pack_tables(synthetic.sensor_for(spec), pipeline_config(args))
    nthreads = os.cpu_count() or 1
    B = frames_np.shape[0]
    # each step = a bounded sample of the workload: as many whole frames as
    # the host does in ~0.5 s (at least one per thread)
    t0 = time.perf_counter()
    oracle.segment_batch(frames_np[:nthreads], packed, nthreads=nthreads)
    per_frame = (time.perf_counter() - t0) / min(nthreads, B) * nthreads
    sample = max(nthreads, min(B, int(0.5 / max(per_frame, 1e-6) * nthreads)))
    for _ in range(args.warmup):
        oracle.segment_batch(frames_np[:sample], packed, nthreads=nthreads)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.segment_batch(frames_np[:sample], packed, nthreads=nthreads)
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    fps = args.steps * sample / tot
    cells = spec.H * spec.W
    line = {
        "impl": "reference", "metric": "frames/s", "value": fps, "unit": "frames/s",
        "points_per_s": fps * cells, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": tot / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded BASELINE generator)",
        "config": workload_config(args, spec, B, 1),
        "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": nthreads, "kind": "port",
                         "sample": f"{sample} of the {B} frames per step, oracle/rangeseg_oracle.c "
                                   f"(reference algorithm restated in C), {nthreads} threads",
                         "why_not_reference": why},
        "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


PER_CONFIG = (   # (label, config id, skip S, core, preset)
    ("c0", 0, 0, False, None), ("c1", 1, 0, False, None), ("c2", 2, 0, False, None),
    ("c3", 3, 0, False, None), ("c4", 4, 0, False, None), ("c1_core", 1, 0, True, None),
    ("c4_core", 4, 0, True, None), ("c1_S1", 1, 1, False, None), ("c1_mc6", 1, 0, False, "mc6"),
    ("c1_mc14", 1, 0, False, "mc14"),
)


def variant_config(core, skip, preset):
    import paper_2003_00575_b200 as rs
    pat = rs.preset_pattern(preset) if preset else rs.skip_pattern(skip)
    if core:
        return rs.PipelineConfig(mc_pattern=pat, ground_removal=False, min_cluster_points=1)
    return rs.PipelineConfig(mc_pattern=pat)


def parity_check(pipe, frames):
    """The fused kernel against the CPU oracle on the same frames: frames whose
    labels / count / sizes differ, and the kernel's OWN edge decisions
    (rs_fast_planes: presence, left, up and Map Connection bits) against the
    oracle's, as a count of differing decisions (north_star's mismatch count)."""
    import numpy as np
    import torch
    from oracle import oracle
    res = pipe.segment_batch(frames)
    host = frames.cpu().numpy()
    wl, wn, ws = oracle.segment_batch(host, pipe.packed, sizes_stride=pipe.sizes_stride)
    torch.cuda.synchronize()
    gl, gn, gs = res.labels.cpu().numpy(), res.n_clusters.cpu().numpy(), res.cluster_sizes.cpu().numpy()
    bad = 0
    for b in range(host.shape[0]):
        k = int(wn[b])
        if gn[b] != wn[b] or not np.array_equal(gl[b], wl[b]) or not np.array_equal(gs[b, :k + 1], ws[b, :k + 1]):
            bad += 1
    out = {"frames_checked": int(host.shape[0]), "label_mismatch_frames": bad}
    if pipe.plan["fast"]:
        planes, _ = pipe.fast_planes(frames)
        want = oracle.planes_batch(host, pipe.packed)
        got = planes.cpu().numpy().view(np.uint32)
        out["edge_decisions_checked"] = int(want.size * 32)
        out["edge_mismatches"] = int(np.unpackbits((got ^ want).view(np.uint8)).sum())
    return out


def time_kernel_graph(pipe, frames, labels, ncl, sizes, steps):
    """Device time of one launch for a batch too small to keep the GPU busy
    from Python: the launch is captured in a CUDA graph and the graph is
    replayed `steps` times between two events (inputs L2-resident: a single
    frame is 0.5 MB)."""
    import torch
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            pipe.segment_batch(frames, labels=labels, n_clusters=ncl, cluster_sizes=sizes)
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        pipe.segment_batch(frames, labels=labels, n_clusters=ncl, cluster_sizes=sizes)
    for _ in range(3):
        g.replay()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(steps):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / steps


def time_kernel(pipe, frames, labels, ncl, sizes, steps, flush, stream):
    import torch
    for _ in range(3):
        pipe.segment_batch(frames, labels=labels, n_clusters=ncl, cluster_sizes=sizes)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    torch.cuda.synchronize()
    for a, b in ev:
        flush.zero_()
        a.record(stream)
        pipe.segment_batch(frames, labels=labels, n_clusters=ncl, cluster_sizes=sizes)
        b.record(stream)
    torch.cuda.synchronize()
    return sum(a.elapsed_time(b) for a, b in ev) / steps


def _plan_of(pipe, batch):
    from paper_2003_00575_b200 import _native
    d = _native.plan_batch(pipe.rs_config, batch)
    return {"rows_per_cta": d["fast_rows"] if d["fast"] else d["dense_rows"],
            "ctas_per_frame": d["fast_ctas"] if d["fast"] else d["dense_ctas"], "fast": bool(d["fast"])}


def per_config_block(args, dev, flush, peak):
    """Every BASELINE config (reference defaults) plus the core / skip /
    Map Connection variants: kernel ms per batch, frames/s, roofline fraction
    (16.5 B/cell + 0.25 per offset) and compulsory fraction (8 B/cell), and
    the parity check of each against the oracle at its full batch."""
    import torch
    import paper_2003_00575_b200 as rs
    from paper_2003_00575_b200 import synthetic
    out = {}
    stream = torch.cuda.current_stream(dev)
    cache = {}
    for label, cid, skip, core, preset in PER_CONFIG:
        spec = synthetic.CONFIGS[cid]
        if cid not in cache:
            cache.clear()
            cache[cid] = synthetic.make_batch(cid, device=dev)
        frames = cache[cid]
        B = frames.shape[0]
        cfg = variant_config(core, skip, preset)
        pipe = rs.Pipeline(synthetic.sensor_for(spec), cfg, device=dev)
        labels = torch.empty((B, spec.H, spec.W), dtype=torch.int32, device=dev)
        ncl = torch.empty((B,), dtype=torch.int32, device=dev)
        sizes = torch.empty((B, pipe.sizes_stride), dtype=torch.int64, device=dev)
        small = B * spec.H * spec.W * 4 < (64 << 20)   # a single frame: launch-bound from Python
        ms = (time_kernel_graph(pipe, frames, labels, ncl, sizes, 200) if small
              else time_kernel(pipe, frames, labels, ncl, sizes, 30, flush, stream))
        cells = B * spec.H * spec.W
        bpc = ALGO_BYTES_PER_CELL + MC_BYTES_PER_OFFSET * len(cfg.mc_pattern)
        e = {"frames": B, "H": spec.H, "W": spec.W, "offsets": len(cfg.mc_pattern),
             "params": ("core" if core else "defaults") + (f", {preset}" if preset else f", S={skip}"),
             "ms": ms, "frames_per_s": B / (ms * 1e-3), "points_per_s": cells / (ms * 1e-3),
             "bytes_per_cell": bpc, "frac": cells * bpc / (ms * 1e-3) / 1e9 / peak,
             "compulsory_frac": cells * COMPULSORY_BYTES_PER_CELL / (ms * 1e-3) / 1e9 / peak,
             "plan": _plan_of(pipe, B),
             "timing": ("CUDA graph replay of the launch, inputs L2-resident (0.5 MB)" if small
                        else "CUDA events per launch, L2 flushed between launches")}
        if not args.no_check:
            e.update(parity_check(pipe, frames))
        out[label] = e
    return out


def per_frame_api(args, dev, n=300):
    """The reference's own per-frame entry (pipeline.py:85-131) through this
    package: Pipeline.segment_range_image on single 64x2048 frames, numpy in
    and numpy out (H2D, kernel, D2H, one sync), wall-clock latency per call."""
    import numpy as np
    import paper_2003_00575_b200 as rs
    from paper_2003_00575_b200 import synthetic
    spec = synthetic.CONFIGS[0]
    frames = synthetic.make_batch(1, 8, device=dev).cpu().numpy()
    pipe = rs.Pipeline(synthetic.sensor_for(spec), rs.PipelineConfig(), device=dev)
    for i in range(10):
        pipe.segment_range_image(frames[i % 8])
    t, k = [], []
    for i in range(n):
        t0 = time.perf_counter()
        _, rec = pipe.segment_range_image(frames[i % 8])
        t.append((time.perf_counter() - t0) * 1e3)
        k.append(rec.ccl)
    t = np.array(t)
    return {"calls": n, "ms_p50": float(np.percentile(t, 50)), "ms_p99": float(np.percentile(t, 99)),
            "ms_mean": float(t.mean()), "kernel_ms_p50": float(np.percentile(k, 50)),
            "frames_per_s": 1e3 / float(t.mean()),
            "path": "Pipeline.segment_range_image(numpy [64, 2048] float32) -> LabelImage; pinned staging, "
                    "rs_segment_batch, one sync; config-0 geometry, reference defaults"}


def eval_path(frames, model):
    """SURVEY.md §8(f)3 on the bench frames: the instance-scoring contingency
    table (rs_contingency, hand-written hash counting) of two segmentations of
    the batch (gt = default labels, pred = core-variant labels), device-timed,
    plus the host matching rules (evaluation.match_instances_batch)."""
    import paper_2003_00575_b200 as rs
    from paper_2003_00575_b200 import evaluation as ev
    import torch
    gt = rs.Pipeline(model, rs.PipelineConfig(), device=frames.device).segment_batch(frames).labels.flatten()
    pred = rs.Pipeline(model, rs.PipelineConfig(ground_removal=False, min_cluster_points=1),
                       device=frames.device).segment_batch(frames).labels.flatten()
    B, n = frames.shape[0], frames[0].numel()
    off = torch.arange(B + 1, dtype=torch.int64, device=frames.device) * n
    ms = ev.contingency_device_ms(gt, pred, off)
    t0 = time.perf_counter()
    out = ev.match_instances_batch(gt, pred, off, ev.EvalConfig(min_gt_points=100))
    match_ms = (time.perf_counter() - t0) * 1e3
    return {"frames": B, "points": B * n, "contingency_device_ms": ms,
            "points_per_s": B * n / (ms * 1e-3), "input_bytes": 8 * B * n,
            "hbm_frac": 8 * B * n / (ms * 1e-3) / 1e9 / measured_peak()[0],
            "match_host_ms": match_ms, "instances_scored": sum(len(o) for o in out),
            "path": "rs_contingency (per-frame shared-memory hash + sort) -> host matching rules"}


def run_b200(args):
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_2003_00575_b200 as rs
    from paper_2003_00575_b200 import synthetic

    rank, local_rank, world = dist_env()
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    spec = synthetic.CONFIGS[args.config]
    B = spec.batch
    frames = synthetic.make_batch(args.config, device=dev, first_seed=rank * B)
    model = synthetic.sensor_for(spec)
    cfg = pipeline_config(args)
    pipe = rs.Pipeline(model, cfg, device=dev, rows_per_cta=args.rows_per_cta)
    labels = torch.empty((B, spec.H, spec.W), dtype=torch.int32, device=dev)
    ncl = torch.empty((B,), dtype=torch.int32, device=dev)
    sizes = torch.empty((B, pipe.sizes_stride), dtype=torch.int64, device=dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        pipe.segment_batch(frames, labels=labels, n_clusters=ncl, cluster_sizes=sizes)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clk:
        wall0 = time.perf_counter()
        for i in range(args.steps):
            flush.zero_()                        # evict L2 between steps
            starts[i].record(stream)
            step()
            ends[i].record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - wall0
    if world > 1:
        dist.barrier()
    kern_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    ms = sum(kern_ms) / len(kern_ms)
    t = torch.tensor([ms], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())

    cells = B * spec.H * spec.W
    fps = world * B / (ms_max * 1e-3)
    algo_bytes = cells * (ALGO_BYTES_PER_CELL + MC_BYTES_PER_OFFSET * len(cfg.mc_pattern))
    peak, peak_src = measured_peak()
    achieved = algo_bytes / (ms * 1e-3) / 1e9

    # ---- end to end through the host-buffer C ABI --------------------------
    e2e = None
    if not args.no_e2e:
        host_in = torch.empty((B, spec.H, spec.W), dtype=torch.float32, pin_memory=True)
        host_in.copy_(frames)
        h_in = host_in.numpy()
        h_lab = torch.empty((B, spec.H, spec.W), dtype=torch.int32, pin_memory=True).numpy()
        h_ncl = torch.empty((B,), dtype=torch.int32, pin_memory=True).numpy()
        h_sz = torch.empty((B, pipe.sizes_stride), dtype=torch.int64, pin_memory=True).numpy()
        for _ in range(max(args.warmup, 3)):
            pipe.segment_batch_host(h_in, h_lab, h_ncl, h_sz)
        if world > 1:
            dist.barrier()
        e_times = []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            pipe.segment_batch_host(h_in, h_lab, h_ncl, h_sz)
            e_times.append(time.perf_counter() - t0)
        te = torch.tensor([sum(e_times) / len(e_times)], device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": world * B / float(te.item()), "unit": "frames/s",
               "h2d_bytes_per_step": int(h_in.nbytes + pipe._tables_host.nbytes),
               "d2h_bytes_per_step": int(h_lab.nbytes + h_ncl.nbytes + h_sz.nbytes),
               "path": "rs_segment_batch_host (C ABI), pinned host buffers, 4 streams, 16 MB chunks"}
        # e2e results must equal the device path
        assert np.array_equal(h_lab, labels.cpu().numpy()), "e2e labels differ from device path"

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    cloud_path = eval_p = None
    if not args.no_cloud and world == 1:
        cloud_path = cloud_bench(args, pipe, frames, spec, flush)
        eval_p = eval_path(frames, model)

    cpu = cpu_port = None
    if not args.no_cpu_baseline:
        done, el = cpu_sample(frames.cpu().numpy(), pipe.packed, args.cpu_seconds, 1)
        cpu_port = {"value": done / el, "unit": "frames/s", "cores": 1, "kind": "port",
                    "sample": f"{done} frames of this workload, single thread, oracle/rangeseg_oracle.c "
                              f"(reference algorithm restated in C), {el:.1f} s"}
        from baseline import ref_bench
        if ref_bench.load()[0] is not None:
            one = ref_bench.single_core(frames[:16].cpu().numpy(), ref_pipe_args(args, spec),
                                        min_seconds=args.cpu_seconds)
            cpu = {"value": one["frames_per_s"], "unit": "frames/s", "cores": 1, "kind": "reference",
                   "sample": f"the workload's first 16 frames, {one['frames_timed']} frame timings; "
                             "rangeseg.bench_run (unmodified reference from baseline/_ref: 1 pinned core, "
                             "GC off, warm-up 3, per-frame TimingRecord.total)",
                   "ms_p50": one["ms_p50"], "ms_p99": one["ms_p99"], "cpu_model": ref_bench.cpu_model(),
                   "host_cores": os.cpu_count()}
        else:
            cpu = cpu_port

    per_config = None
    if not args.no_per_config and world == 1:
        per_config = per_config_block(args, dev, flush, peak)
    frame_api = per_frame_api(args, dev) if world == 1 and not args.no_frame_api else None
    check = None
    if not args.no_check:
        check = parity_check(pipe, frames)

    traffic = None
    tf = ROOT / "profiles" / "kernel_traffic.json"
    if tf.exists():
        try:
            traffic = json.loads(tf.read_text()).get(f"config{args.config}" + ("_core" if args.core else "")
                                                     + (f"_S{args.skip}" if args.skip else ""))
        except Exception:
            traffic = None

    line = {
        "metric": "frames/s", "value": fps, "unit": "frames/s",
        "points_per_s": fps * spec.H * spec.W,
        "valid_points_per_s": fps * float((frames > 0).float().mean()) * spec.H * spec.W,
        "n_gpus": world, "steps": args.steps, "warmup": max(args.warmup, 3),
        "ms_per_step": ms_max, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded BASELINE generator)",
        "config": workload_config(args, spec, B, world),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "algorithmic_bytes_per_launch": algo_bytes,
                     "bytes_per_cell": algo_bytes / cells,
                     "compulsory_frac": cells * COMPULSORY_BYTES_PER_CELL / (ms * 1e-3) / 1e9 / peak,
                     "peak_source": peak_src, "kernel": "rs_fast_kernel (one launch per step; node-capacity overflow handled in-kernel)",
                     "kernel_ms": ms},
        "cpu_baseline": cpu,
        "cpu_baseline_port": cpu_port,
        "e2e": e2e,
        "edge_mismatches": None if check is None else check.get("edge_mismatches"),
        "frames_checked": None if check is None else check["frames_checked"],
        "parity": check,
        "per_frame_api": frame_api,
        "per_config": per_config,
        "cloud_path": cloud_path,
        "eval_path": eval_p,
        "gpu_launches": args.steps,   # one rs_fast_kernel (or rs_dense_kernel) launch per step
        "clocks": clk.summary(),
        "wall_s_timed_region": wall,
        "plan": {"rows_per_cta": pipe.rows_per_cta, "ctas_per_frame": pipe.ctas_per_frame,
                 "smem_bytes": pipe.smem_bytes},
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
