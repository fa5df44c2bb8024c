"""Timing harness for the UNMODIFIED reference (rangeseg, pure Python + numba)
installed in baseline/_ref by baseline/install.sh.

The reference's own CPU path is called through its public API only:
``rangeseg.Pipeline(SensorModel(...), PipelineConfig(...)).segment_range_image``
(/root/reference/pkg/src/rangeseg/pipeline.py:85-131), timed two ways, as
BASELINE.md's CPU-baseline plan asks:

* ``single_core``: the reference's ``bench_run`` (pipeline.py:274-311): pinned
  to one core, GC off, 3 warm-up frames, per-frame ``TimingRecord.total``
  (excludes I/O and generation);
* ``all_cores``: one process per host core (the GIL makes threads useless,
  pipeline.py:170-197), each holding its own ``Pipeline`` pinned to its core,
  wall clock over every process's share of the sample.

Nothing of this repository's product package is on that path; the frames are
the same seeded synthetic BASELINE frames the GPU arm segments.
"""

from __future__ import annotations

import multiprocessing as mp
import os
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF_DIR = HERE / "_ref"


def load():
    """The installed reference package, or None (with the reason)."""
    if not (REF_DIR / "rangeseg").is_dir():
        return None, f"{REF_DIR} missing (run baseline/install.sh)"
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/rangeseg_numba_cache")
    if str(REF_DIR) not in sys.path:
        sys.path.insert(0, str(REF_DIR))
    try:
        import rangeseg
    except Exception as e:   # numba missing, ...
        return None, f"import rangeseg failed: {e!r}"
    return rangeseg, None


def make_pipeline(rangeseg, H, W, top_deg, bottom_deg, mount, offsets=(), ground=True, min_points=100):
    """Reference objects for a BASELINE geometry (uniform linspace channels over a
    full revolution, the same construction as SensorModel.fov / the configs)."""
    model = rangeseg.SensorModel(np.linspace(top_deg, bottom_deg, H), 360.0 / W, mount, width=W)
    cfg = rangeseg.PipelineConfig(mc_pattern=rangeseg.MCPattern(tuple(tuple(o) for o in offsets)),
                                  ground_removal=bool(ground), min_cluster_points=int(min_points))
    return rangeseg.Pipeline(model, cfg)


def single_core(frames, pipe_args, min_seconds=5.0):
    """bench_run semantics on one pinned core: frames/s = 1000 / mean per-frame ms."""
    rangeseg, why = load()
    if rangeseg is None:
        raise RuntimeError(why)
    pipe = make_pipeline(rangeseg, **pipe_args)
    recs = list(rangeseg.bench_run(list(frames), pipe, repetitions=1, warmup=3).records)
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < min_seconds:
        recs += list(rangeseg.bench_run(list(frames), pipe, repetitions=1, warmup=0).records)
    tot = np.array([r.total for r in recs])
    return {"frames_per_s": 1000.0 / float(tot.mean()), "ms_mean": float(tot.mean()),
            "ms_p50": float(np.percentile(tot, 50)), "ms_p99": float(np.percentile(tot, 99)),
            "frames_timed": int(tot.size), "distinct_frames": int(len(frames))}


# ------------------------------------------------------------ all cores ------
_W = {}


def _init(frames, pipe_args, counter):
    with counter.get_lock():
        idx = counter.value
        counter.value += 1
    cores = sorted(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else []
    if cores:
        try:
            os.sched_setaffinity(0, {cores[idx % len(cores)]})
        except OSError:
            pass
    import gc
    gc.disable()
    rangeseg, why = load()
    if rangeseg is None:
        raise RuntimeError(why)
    _W["pipe"] = make_pipeline(rangeseg, **pipe_args)
    _W["frames"] = [rangeseg.from_ranges(f) for f in frames]
    for ri in _W["frames"][:3]:   # warm-up: numba JIT / cache load
        _W["pipe"].segment_range_image(ri)


def _work(n):
    fr = _W["frames"]
    pipe = _W["pipe"]
    for i in range(n):
        pipe.segment_range_image(fr[i % len(fr)])
    return n


class AllCores:
    """One reference process per host core; ``step()`` = every process
    segments ``per_proc`` frames, timed by wall clock."""

    def __init__(self, frames, pipe_args, nproc=None):
        self.nproc = nproc or os.cpu_count() or 1
        ctx = mp.get_context("fork")
        counter = ctx.Value("i", 0)
        self.pool = ctx.Pool(self.nproc, initializer=_init, initargs=(frames, pipe_args, counter))
        self.pool.map(_work, [1] * self.nproc, chunksize=1)   # every worker initialised

    def step(self, per_proc):
        t0 = time.perf_counter()
        done = sum(self.pool.map(_work, [per_proc] * self.nproc, chunksize=1))
        return done, time.perf_counter() - t0

    def close(self):
        self.pool.close()
        self.pool.join()


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"
