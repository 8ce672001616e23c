#!/usr/bin/env python
"""Benchmark of the NIRC hot path on B200 (BASELINE.json).

Workload (config 2, the isolated NIRC inference micro-bench, which is what
BASELINE.json's query-rate metric is quoted on and fits one GPU): 2^22
random (pos, dir) queries per GPU, default 12-level hash grid + 4-band SH,
64-wide 2-hidden-layer MLP, theta = init_theta(make_spec(depth=2), seed=1,
out_scale=0.1).  One step = one fused encode + tcgen05 MLP pass
(``full_forward`` / C-ABI ``nirc_full_forward``) over the whole batch with
inputs resident in HBM.  Inputs (2^22 x 104 B = 436 MB of f64 SoA rows) are
larger than L2, so no explicit flush is needed between steps; the 3 MB hash
tables are L2-resident by design.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

Prints ONE JSON line on rank 0.  Multi-GPU: one process per GPU (torchrun),
each rank processes its own 2^22 queries (weak scaling, no collective on
the data path -- the query stream shards with no exchange); timing is the
max over ranks of the device time.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_QUERIES = 1 << 22
DEPTH = 2
# algorithmic work per query
FLOPS_PER_QUERY = 2 * (47 * 64 + 64 * 64 + 64 * 3)     # 14,592 for D = 2
HBM_BYTES_PER_QUERY = 13 * 8 + 3 * 4                  # f64 rows in + f32 rgb out = 116
L2_GATHER_BYTES_PER_QUERY = 12 * 8 * 2 * 4            # 768
PRECISION = int(os.environ.get("NIRC_BENCH_PRECISION", "2"))  # 2: tcgen05 2xFP16 split


def cfg2_config(world):
    """The workload dict both arms print (the driver compares them)."""
    return {"workload": "cfg2 NIRC inference micro-bench: 2^22 random (pos,dir) queries per "
                        "GPU, fused hash-grid+SH encode + 64-wide 2-hidden-layer MLP",
            "model": "nirc 12x2^15x2 hash + SH4 + 64x2 MLP", "global_batch": world * N_QUERIES,
            "seq_len": 1, "parallelism": f"dp{world} (independent query shards)",
            "l2_flush": "inputs (436 MB/step) larger than L2; hash tables L2-resident"}


def host_info():
    """The CPU baseline's context: CPU model, threads, and the
    numpy / numba / OpenBLAS versions of the reference's stack."""
    info = {"cpu_model": None, "host_threads": os.cpu_count()}
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                info["cpu_model"] = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    try:
        import numpy
        info["numpy"] = numpy.__version__
    except Exception:
        info["numpy"] = None
    try:
        import numba
        info["numba"] = numba.__version__
    except Exception:
        info["numba"] = None
    try:
        import threadpoolctl
        blas = [d for d in threadpoolctl.threadpool_info() if d.get("user_api") == "blas"]
        info["openblas"] = (blas[0].get("internal_api", "") + " " + blas[0].get("version", "")
                            + " " + str(blas[0].get("architecture", ""))) if blas else None
    except Exception:
        info["openblas"] = None
    return info


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--n", type=int, default=N_QUERIES)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-frame", action="store_true")
    ap.add_argument("--no-extra-frames", action="store_true")
    ap.add_argument("--frame-steps", type=int, default=10)
    return ap.parse_args()


# ------------------------------------------------------------- clocks ----
class ClockSampler:
    """Samples SM clock + throttle reasons via NVML during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, index, period=0.005):
        self.samples, self.reasons = [], 0
        self.max_mhz = None
        self._stop = threading.Event()
        self.period = period
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nv is not None:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv is not None:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        s = sorted(self.samples)
        names = [n for b, n in self.REASONS.items() if self.reasons & b and n != "gpu_idle"]
        return {"sm_mhz": s[len(s) // 2], "sm_max_mhz": self.max_mhz, "reasons": names,
                "samples": len(s)}


# ------------------------------------------------------------ CPU legs ---
def _oracle_chunk(args):
    n, seed = args
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import nirc_oracle as O

    spec = O.Spec(depth=DEPTH)
    theta = O.init_theta(spec, seed=1, out_scale=0.1)
    q = O.measure_queries(n, seed=seed)
    t0 = time.perf_counter()
    O.full_forward(spec, theta, *q)
    return n, time.perf_counter() - t0


def cpu_baseline(cores=1, chunks=None, chunk=1 << 15, pool=None):
    """The oracle port (encode_batch + mlp_forward in numpy, the reference's
    own batch algorithm) on the host cores: `chunks` chunks of 2^15 queries.
    With cores > 1 the chunks run on a process pool (one chunk per core)."""
    chunks = chunks or max(4, 2 * cores)
    jobs = [(chunk, 100 + i) for i in range(chunks)]
    t0 = time.perf_counter()
    if cores == 1:
        res = [_oracle_chunk(j) for j in jobs]
    else:
        res = pool.map(_oracle_chunk, jobs)
    wall = time.perf_counter() - t0
    n = sum(r[0] for r in res)
    if cores == 1:
        rate = n / sum(r[1] for r in res)
    else:
        rate = n / wall
    return rate, n


def run_reference(args, rank, world):
    """The reference arm (tier rules): the reference's CPU algorithm for the
    path -- the oracle port, a numpy restatement of encode_batch +
    mlp_forward -- on every host core (one process per core, one 2^15-query
    chunk per core per step)."""
    if rank != 0:
        return
    import multiprocessing as mp

    cores = os.cpu_count() or 1
    times = []
    nq = 0
    with mp.get_context("spawn").Pool(cores) as pool:
        pool.map(_oracle_chunk, [(64, 1)] * cores)  # import + first-touch outside the timing
        for s in range(args.warmup + args.steps):
            rate, n = cpu_baseline(cores=cores, chunks=cores, chunk=1 << 15, pool=pool)
            if s >= args.warmup:
                times.append(n / rate)
                nq += n
    value = nq / sum(times)
    line = {
        "impl": "reference", "metric": "nirc_queries_per_sec", "value": value,
        "unit": "queries/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * sum(times) / len(times), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": cfg2_config(args.gpus),
        "cpu_baseline": {"value": value, "unit": "queries/s", "cores": cores, "kind": "port",
                         "sample": f"{cores} x 2^15 random queries per step (one process per "
                                   "core) through oracle/nirc_oracle.full_forward (numpy "
                                   "restatement of encode_batch + mlp_forward)",
                         "host": host_info()},
        "e2e": {"value": value, "unit": "queries/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------- frame leg -------
FLOPS_PER_QUERY_D4 = 2 * (47 * 64 + 3 * 64 * 64 + 64 * 3)  # 30,976: the frame caches' D = 4


def infer_roofline(queries, infer_ms):
    """The frame inference kernel against the tensor roofline: useful
    (reference-arithmetic) FLOP per launch / its device time, over the
    measured dense bf16 peak; the 2xFP16 split issues 3 MMAs per product."""
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    peak = float(peaks.get("bf16_tflops", 1590.0))
    tf = queries * FLOPS_PER_QUERY_D4 / (infer_ms * 1e-3) / 1e12
    return {"bound": "tensor", "kernel": "k_infer_ws (fused encode + tcgen05 MLP + MLMC combine)",
            "useful_flop_per_launch": queries * FLOPS_PER_QUERY_D4, "avg_launch_ms": infer_ms,
            "achieved": tf, "peak": peak, "unit": "TFLOP/s", "frac": tf / peak,
            "issued_frac": 3 * tf / peak,
            "peak_source": "MEASURED_PEAKS.json bf16_tflops" if peaks else "fallback",
            "timing": "CUDA events on the render stream around the launch (C-ABI stage timer), "
                      "sequential frame (no train-stream overlap), median over frames"}


def frame_bench(frames, warmup, width=1920, height=1080, nc=(16,), comm=None, name="cfg3"):
    """BASELINE config 3: Cornell at 1920x1080, two-level with nc=(16,) at
    the first cache vertex, spp 1, D = 4 cache; then collect ceil(0.025 W H)
    training paths and 4 Adam steps of 16384 records.  Device time per
    phase with CUDA events; frames after `warmup` are timed.  With a
    multi-rank `comm` the frame is sharded (distributed.py: pixel-row bands,
    path shards + record all-gather, tile shards + gradient all-reduce) and
    each phase time is the max over ranks."""
    import torch

    from paper_2412_04634_b200 import distributed as D
    from paper_2412_04634_b200.caches import Cache, default_train_count, train_frame
    from paper_2412_04634_b200.estimators import render_and_collect
    from paper_2412_04634_b200.frame import config3
    from paper_2412_04634_b200.scene import load_builtin

    scene = load_builtin("cornell").with_resolution(width, height)
    cache = Cache.create("nirc", scene, seed=0, init="random")
    cfg = config3(nc)
    stream = torch.cuda.current_stream()
    phases = {"render": [], "collect": [], "train": [], "frame": []}
    queries, records = [], []
    count = default_train_count(scene)
    world = comm.world if comm is not None else 1
    ops = D.DeviceOps() if world > 1 else None
    # per-stage device times of the render launch set (C-ABI stage events)
    import ctypes

    from paper_2412_04634_b200 import _lib

    lib = _lib.load()
    lib.nirc_stage_timing(1)
    stage_buf = (ctypes.c_float * 3)()
    stages = {"trace": [], "infer": [], "accumulate": []}
    for f in range(warmup + frames):
        if comm is not None:
            comm.barrier()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        ev[0].record(stream)
        # render + training walks of the frame in one trace launch (the
        # record all-gather of the multi-GPU frame is inside "collect")
        if world > 1:
            rows = D.split_range(height, world, comm.rank)
            paths = D.split_range(count, world, comm.rank)
            _, _, _, q, local = render_and_collect(scene, cfg, cache, seed=0, spp=1, frame=f,
                                                   count=count, rows=rows, paths=paths)
        else:
            _, _, _, q, rec = render_and_collect(scene, cfg, cache, seed=0, spp=1, frame=f,
                                                 count=count)
        ev[1].record(stream)
        if world > 1:
            packed = D.pack_records({k: getattr(local, k) for k, _ in D.REC_COLS})
            rec = D.unpack_records(comm.all_gather_rows(packed), cache.record_kind, f)
        ev[2].record(stream)
        if world > 1:
            D.train_frame_sharded(cache, rec, comm, steps=4, ops=ops)
        else:
            train_frame(cache, rec, steps=4)
        ev[3].record(stream)
        torch.cuda.synchronize()
        if f >= warmup:
            _lib.check(lib.nirc_stage_times(stage_buf, 3), "nirc_stage_times")
            for k, v in zip(("trace", "infer", "accumulate"), stage_buf):
                stages[k].append(float(v))
            t = torch.tensor([ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2]),
                              ev[2].elapsed_time(ev[3]), ev[0].elapsed_time(ev[3])],
                             device="cuda")
            if comm is not None:
                comm.all_reduce_max_(t)
            t = t.tolist()
            for k, v in zip(("render", "collect", "train", "frame"), t):
                phases[k].append(v)
            qt = q.clone()
            if comm is not None:
                comm.all_reduce_sum_(qt)
            queries.append(int(qt.item()))
            records.append(len(rec))
    lib.nirc_stage_timing(0)
    if world > 1:
        same = D.replicas_identical(cache, comm)
    else:
        same = True
    med = {k: sorted(v)[len(v) // 2] for k, v in phases.items()}
    smed = {k: sorted(v)[len(v) // 2] for k, v in stages.items()}
    return {
        "metric": f"ms_per_frame_{width}x{height}", "value": med["frame"], "unit": "ms/frame",
        "higher_is_better": False, "frames": frames, "warmup": warmup, "n_gpus": world,
        "render_collect_ms": med["render"], "record_allgather_ms": med["collect"],
        "train_ms": med["train"],
        "queries_per_frame": queries[-1], "records_per_frame": records[-1],
        "train_paths_per_frame": count,
        "train_samples_per_sec": 4 * min(16384, records[-1]) / (med["train"] * 1e-3),
        "render_queries_per_sec": queries[-1] / (med["render"] * 1e-3),
        "stage_ms": {k + "_ms": v for k, v in smed.items()},
        "infer_roofline": infer_roofline(queries[-1] // world, smed["infer"]),
        "phases": "render_collect = one nirc_render_collect launch set (path tracer with the "
                  "training walks as its first work items, fused inference, accumulation, "
                  "record compaction); record_allgather = multi-GPU record exchange",
        "replicas_identical": same,
        "config": f"{name}: cornell {width}x{height}, two-level nc={tuple(nc)}, spp 1, D=4 "
                  f"cache, collect {count:,} paths, 4 x min(16384, records) train steps"
                  + (f"; sharded over {world} GPUs (row bands, path shards, "
                     "NCCL gradient all-reduce)" if world > 1 else ""),
        "reference_cpu_context": "SURVEY.md 6: 122.6 s/frame on 1 core (not re-timed here)",
    }


def frame_bench_overlap(frames, warmup, width=1920, height=1080, nc=(16,), name="cfg3"):
    """The same frame as frame_bench on one GPU through frame.FramePipeline:
    render(f) (+ the walks collecting frame f+1's records) on the render
    stream while train(f) runs on a second stream against a theta_f snapshot
    (SURVEY.md 8(e)).  Frame time = device time from the frame's start on
    the render stream to the later of the two streams' ends (CUDA events)."""
    import torch

    from paper_2412_04634_b200.caches import Cache
    from paper_2412_04634_b200.frame import FramePipeline, config3
    from paper_2412_04634_b200.scene import load_builtin

    scene = load_builtin("cornell").with_resolution(width, height)
    cache = Cache.create("nirc", scene, seed=0, init="random")
    pipe = FramePipeline(scene, cache, config3(nc), seed=0)
    frame_ms, render_ms, train_ms, queries, records = [], [], [], [], []
    for f in range(warmup + frames):
        e0, er = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(pipe.s_render)
        _, st = pipe.step(f)
        er.record(pipe.s_render)
        torch.cuda.synchronize()
        if f >= warmup:
            r = e0.elapsed_time(er)
            t = 0.0
            end = r
            if pipe.train_events is not None:
                t0, t1 = pipe.train_events
                t = t0.elapsed_time(t1)
                end = max(r, e0.elapsed_time(t1))
            frame_ms.append(end)
            render_ms.append(r)
            train_ms.append(t)
            queries.append(st.queries)
            records.append(st.records)
    med = lambda v: sorted(v)[len(v) // 2]  # noqa: E731
    return {
        "metric": f"ms_per_frame_{width}x{height}", "value": med(frame_ms), "unit": "ms/frame",
        "higher_is_better": False, "frames": frames, "warmup": warmup, "n_gpus": 1,
        "render_collect_ms": med(render_ms), "train_stream_span_ms": med(train_ms),
        "queries_per_frame": queries[-1], "records_per_frame": records[-1],
        "render_queries_per_sec": queries[-1] / (med(render_ms) * 1e-3),
        "phases": "render_collect = the render stream (snapshot copy, one nirc_render_collect "
                  "launch set: path tracer with the NEXT frame's training walks as its first "
                  "work items, fused inference, accumulation, record compaction); "
                  "train_stream_span = first to last event of the train stream (4 steps on "
                  "this frame's records), which shares the SMs with the render stream -- its "
                  "kernels' own time is the sequential leg's train_ms",
        "overlap": True,
        "config": f"{name}: cornell {width}x{height}, two-level nc={tuple(nc)}, spp 1, D=4 "
                  f"cache, collect 0.025 W H paths, 4 x min(16384, records) train steps; "
                  "render(f) || train(f) (frame.FramePipeline)",
        "reference_cpu_context": "SURVEY.md 6: 122.6 s/frame on 1 core (not re-timed here)",
    }


def frame_bench_sharded(frames, warmup, comm, width=1920, height=1080, nc=(16,), name="cfg3"):
    """The sharded frame (N > 1) through distributed.ShardedFramePipeline:
    render(f) of this rank's row band (+ its share of frame f+1's training
    walks) on the render stream while the record all-gather and the
    tile-sharded train(f) with one gradient all-reduce per step run on a
    second stream.  Frame time per rank = device time from the frame's
    start to the later stream's end; the max over ranks is reported."""
    import torch

    from paper_2412_04634_b200 import distributed as D
    from paper_2412_04634_b200.caches import Cache
    from paper_2412_04634_b200.frame import config3
    from paper_2412_04634_b200.scene import load_builtin

    scene = load_builtin("cornell").with_resolution(width, height)
    cache = Cache.create("nirc", scene, seed=0, init="random")
    pipe = D.ShardedFramePipeline(scene, cache, config3(nc), comm, seed=0)
    frame_ms, render_ms, train_ms, queries, records = [], [], [], [], []
    for f in range(warmup + frames):
        comm.barrier()
        torch.cuda.synchronize()
        e0, er = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(pipe.s_render)
        _, rows, st = pipe.step(f)
        er.record(pipe.s_render)
        torch.cuda.synchronize()
        if f >= warmup:
            t0, t1 = pipe.train_events
            t = torch.tensor([max(e0.elapsed_time(er), e0.elapsed_time(t1)),
                              e0.elapsed_time(er), t0.elapsed_time(t1)], device="cuda")
            comm.all_reduce_max_(t)
            q = st["queries"].clone()
            comm.all_reduce_sum_(q)
            a, b, c = t.tolist()
            frame_ms.append(a)
            render_ms.append(b)
            train_ms.append(c)
            queries.append(int(q.item()))
            records.append(st.get("records", 0))
    same = D.replicas_identical(cache, comm)
    med = lambda v: sorted(v)[len(v) // 2]  # noqa: E731
    return {
        "metric": f"ms_per_frame_{width}x{height}", "value": med(frame_ms), "unit": "ms/frame",
        "higher_is_better": False, "frames": frames, "warmup": warmup, "n_gpus": comm.world,
        "render_collect_ms": med(render_ms), "train_stream_span_ms": med(train_ms),
        "queries_per_frame": queries[-1], "records_per_frame": records[-1],
        "render_queries_per_sec": queries[-1] / (med(render_ms) * 1e-3),
        "replicas_identical": same, "overlap": True,
        "phases": "per rank: render_collect = its row band + its share of the next frame's "
                  "walks (render stream); train_stream_span = record all-gather + 4 sharded "
                  "steps with one gradient all-reduce each (train stream); max over ranks",
        "config": f"{name}: cornell {width}x{height}, two-level nc={tuple(nc)}, spp 1, D=4 "
                  f"cache, collect 0.025 W H paths, 4 x min(16384, records) train steps; "
                  f"sharded over {comm.world} GPUs (row bands, path shards, tile shards) with "
                  "render(f) || train(f) (distributed.ShardedFramePipeline)",
        "reference_cpu_context": "SURVEY.md 6: 122.6 s/frame on 1 core (not re-timed here)",
    }


def convergence_bench(frames=100, width=1920, height=1080, ref_spp=64):
    """BASELINE config 4: the teleport scene (its lamp jumps at frame 40) at
    1920x1080, `frames` frames of continuous online training with the cfg3
    estimator ("as cfg 3 per frame") through the device frame
    loop (frame.FramePipeline: experiment.py:149-185's render / collect / train
    with render(f) || train(f)),
    MRSE per frame against a ref_spp device-PT reference of each geometry
    state (experiment.py's _ReferenceBank), computed on the device."""
    import torch

    from paper_2412_04634_b200.config import RunConfig
    from paper_2412_04634_b200.estimators import EstimatorConfig, render_device
    from paper_2412_04634_b200.experiment import REF_SEED_OFFSET, _make_cache
    from paper_2412_04634_b200.frame import FramePipeline, config3
    from paper_2412_04634_b200.scene import load_builtin

    rc = RunConfig(scene="teleport", mode="two-level", nc=(16,), max_cache_vertices=1,
                   frames=frames, seed=0, ref_spp=ref_spp)
    scene = load_builtin("teleport").with_resolution(width, height)
    cache = _make_cache(rc, scene)
    est = config3((16,))
    pipe = FramePipeline(scene, cache, est, rc.seed)
    stream = pipe.s_render
    refs, ref_ms = {}, 0.0
    ms, mrse = [], []
    for f in range(frames):
        scene = scene.at_frame(f)
        key = scene.content_hash()
        if key not in refs:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            img, _, _, _ = render_device(scene, EstimatorConfig(mode="pt"), None,
                                         rc.seed + REF_SEED_OFFSET, ref_spp, 0)
            e1.record(stream)
            torch.cuda.synchronize()
            ref_ms += e0.elapsed_time(e1)
            refs[key] = img / ref_spp
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        (img, _, _), _ = pipe.step(f)
        stream.wait_stream(pipe.s_train)
        e1.record(stream)
        ref = refs[key]
        mrse.append(torch.mean((img - ref) ** 2 / (ref * ref + 0.01)))
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    m = [float(x.item()) for x in mrse]
    # plain 1-spp PT on the same frames and pixels: what the cache buys
    pt = []
    for f in range(frames - 10, frames):
        img, _, _, _ = render_device(scene.at_frame(f), EstimatorConfig(mode="pt"), None,
                                     rc.seed, 1, f)
        ref = refs[scene.at_frame(f).content_hash()]
        pt.append(float(torch.mean((img - ref) ** 2 / (ref * ref + 0.01)).item()))

    def win(lo, hi):
        return sum(m[lo:hi]) / max(1, len(m[lo:hi]))

    return {
        "metric": f"ms_per_frame_{width}x{height}_teleport_{frames}f", "unit": "ms/frame",
        "value": sorted(ms)[len(ms) // 2], "mean_ms": sum(ms) / len(ms),
        "higher_is_better": False, "frames": frames, "n_gpus": 1,
        "mrse_frame0": m[0], "mrse_mean_30_40": win(30, 40), "mrse_mean_40_50": win(40, 50),
        "mrse_mean_last10": win(frames - 10, frames), "mrse_final": m[-1],
        "pt_mrse_mean_last10": sum(pt) / len(pt),
        "reference": f"device PT, {ref_spp} spp per geometry state ({len(refs)} states, "
                     f"{ref_ms:.0f} ms, not in the frame time)",
        "config": "cfg4: teleport 1920x1080 (lamp jumps at frame 40), two-level nc=(16,), "
                  "spp 1, D=4 cache (zero-initialised output layer), collect 0.025 W H paths, "
                  "4 Adam steps per frame; MRSE = mean((img-ref)^2/(ref^2+0.01)) "
                  "(metrics.py) on the device",
    }


# ------------------------------------------------------------ GPU leg ----
def run_b200(args, rank, world, local_rank):
    import numpy as np
    import torch

    torch.cuda.set_device(local_rank % torch.cuda.device_count())
    dist = None
    if world > 1:
        import torch.distributed as dist

    from paper_2412_04634_b200 import _dev, _lib
    from paper_2412_04634_b200.mlp import full_forward, init_theta, make_spec
    from paper_2412_04634_b200 import workloads

    lib = _lib.load()
    n = args.n
    spec = make_spec(depth=DEPTH)
    theta = torch.from_numpy(init_theta(spec, seed=1, out_scale=0.1)).cuda()
    q_dev = workloads.measure_queries_device(n, seed=rank)
    Y = torch.empty((n, 3), dtype=torch.float32, device="cuda")
    cs = _lib.make_c_spec(spec)
    ptrs = [_dev.ptr(a) for a in q_dev]
    stream = torch.cuda.current_stream()

    flags = torch.zeros(1, dtype=torch.int32, device="cuda")

    def step():
        _lib.check(lib.nirc_full_forward(cs, _dev.ptr(theta), *ptrs, n, _dev.ptr(Y), PRECISION,
                                         _dev.ptr(flags), _dev.stream()), "nirc_full_forward")

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    barrier()
    # ---- timed region: K steps, device events on the launching stream ----
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * args.steps)]
    with ClockSampler(local_rank) as clocks:
        barrier()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for k in range(args.steps):
            ev[2 * k].record(stream)
            step()
            ev[2 * k + 1].record(stream)
        t1.record(stream)
        barrier()
    ms = t0.elapsed_time(t1)
    per_launch = [ev[2 * k].elapsed_time(ev[2 * k + 1]) for k in range(args.steps)]
    ms_t = torch.tensor([ms], device="cuda")
    if dist is not None:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms = float(ms_t.item())
    value = world * n * args.steps / (ms * 1e-3)

    # ---- end-to-end through the public API with pinned host buffers ----
    # the user's call: pinned host f64 rows in, host f32 rgb out; full_forward
    # streams them through its chunked H2D / kernel / D2H pipeline
    host = [torch.from_numpy(np.ascontiguousarray(a.cpu().numpy())).pin_memory() for a in q_dev]
    y_host = torch.empty((n, 3), dtype=torch.float32).pin_memory()
    e2e_steps = max(3, min(args.steps, 40))
    y_last = [None]

    def e2e_step():
        y_last[0] = full_forward(spec, theta, *host, precision=PRECISION, out=y_host)

    for _ in range(2):
        e2e_step()
    barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    eps_ = [torch.cuda.Event(enable_timing=True) for _ in range(e2e_steps + 1)]
    e0.record(stream)
    eps_[0].record(stream)
    for k in range(e2e_steps):
        e2e_step()
        eps_[k + 1].record(stream)
    e1.record(stream)
    barrier()
    e2e_per_step = sorted(eps_[k].elapsed_time(eps_[k + 1]) for k in range(e2e_steps))
    e_ms = torch.tensor([e0.elapsed_time(e1)], device="cuda")
    if dist is not None:
        dist.all_reduce(e_ms, op=dist.ReduceOp.MAX)
    e2e_value = world * n * e2e_steps / (float(e_ms.item()) * 1e-3)
    h2d = int(sum(h.numel() * h.element_size() for h in host))
    d2h = int(y_last[0].numel() * 4)

    # ---- the same call as a numpy user makes it (the reference's types):
    # numpy theta and numpy f64 rows in (pageable), numpy f32 rgb out; the
    # call returns host results, so its wall time is the step time
    host_np = [h.numpy() for h in host]
    theta_np = theta.cpu().numpy()
    full_forward(spec, theta_np, *host_np, precision=PRECISION)
    np_steps = 5
    barrier()
    t0w = time.perf_counter()
    for _ in range(np_steps):
        y_np = full_forward(spec, theta_np, *host_np, precision=PRECISION)
    np_s = time.perf_counter() - t0w
    assert isinstance(y_np, np.ndarray)
    # the PCIe roofline of the pinned e2e path: the same bytes as plain pinned
    # copies (H2D of the five input columns while D2H of the outputs runs on
    # a second stream), CUDA events, best of 3
    pcie_ms = []
    d_in = [torch.empty_like(h, device="cuda") for h in host]
    d_out = torch.empty((n, 3), dtype=torch.float32, device="cuda")
    s_d2h = torch.cuda.Stream()
    for _ in range(3):
        barrier()
        p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        p0.record(stream)
        s_d2h.wait_stream(stream)
        with torch.cuda.stream(s_d2h):
            y_host.copy_(d_out, non_blocking=True)
        for d, h in zip(d_in, host):
            d.copy_(h, non_blocking=True)
        stream.wait_stream(s_d2h)
        p1.record(stream)
        torch.cuda.synchronize()
        pcie_ms.append(p0.elapsed_time(p1))
    del d_in, d_out
    pcie_best = min(pcie_ms)
    e2e_pcie = {"copy_only_ms": pcie_best,
                "h2d_gbs": h2d / (pcie_best * 1e-3) / 1e9,
                "e2e_frac_of_copy_only": (pcie_best * 1e-3) / (float(e_ms.item()) * 1e-3
                                                               / e2e_steps),
                "note": "the pinned e2e step against copying the same bytes alone: its bound"}
    e2e_numpy = {"value": world * n * np_steps / np_s, "unit": "queries/s", "steps": np_steps,
                 "h2d_bytes_per_step": h2d + theta_np.nbytes, "d2h_bytes_per_step": d2h,
                 "path": "paper_2412_04634_b200.mlp.full_forward on numpy arrays (pageable host "
                         "memory, numpy theta), host wall clock per call"}

    fb = None
    if not args.no_frame:
        from paper_2412_04634_b200 import distributed as D

        comm = D.Comm() if world > 1 else None
        if world == 1:
            # one GPU: render(f) || train(f) (frame.FramePipeline); the
            # sequential loop's numbers ride along for comparison
            fb = frame_bench_overlap(args.frame_steps, 3)
            fb["sequential"] = frame_bench(args.frame_steps, 3)
        else:
            fb = frame_bench_sharded(args.frame_steps, 3, comm)
            fb["sequential"] = frame_bench(args.frame_steps, 3, comm=comm)
        if not args.no_extra_frames:
            # BASELINE cfg5 (4K, 32 NIRC samples/pixel as nc=(16,16): the
            # reference caps N_c at 28 per vertex) and cfg1 (the reference's
            # CPU-runnable 128^2 frame), both sharded like cfg3 when N > 1
            if world == 1:
                fb["cfg5_4k"] = frame_bench_overlap(max(3, args.frame_steps // 2), 2, 3840,
                                                    2160, (16, 16), name="cfg5")
                fb["cfg1_128"] = frame_bench_overlap(args.frame_steps, 3, 128, 128, (8,),
                                                     name="cfg1")
            else:
                fb["cfg5_4k"] = frame_bench_sharded(max(3, args.frame_steps // 2), 2, comm, 3840,
                                                    2160, (16, 16), name="cfg5")
                fb["cfg1_128"] = frame_bench_sharded(args.frame_steps, 3, comm, 128, 128, (8,),
                                                     name="cfg1")
            fb["cfg1_128"]["reference_cpu_context"] = (
                "SURVEY.md 6: 1.28 s/frame for cfg1 on 1 core (render 1084 + collect 12 + "
                "train 179 ms)")
        if world == 1 and not args.no_extra_frames:
            fb["cfg4_teleport_1080p"] = convergence_bench()
    if rank != 0:
        return
    import json as _json

    peaks = {}
    try:
        peaks = _json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    avg_launch_ms = sum(per_launch) / len(per_launch)
    achieved_gbs = n * HBM_BYTES_PER_QUERY / (avg_launch_ms * 1e-3) / 1e9
    tflops = n * FLOPS_PER_QUERY / (avg_launch_ms * 1e-3) / 1e12
    l2_gbs = n * L2_GATHER_BYTES_PER_QUERY / (avg_launch_ms * 1e-3) / 1e9
    traffic = None
    prof = {}
    try:
        prof = _json.load(open(os.path.join(ROOT, "profiles", "full_forward_traffic.json")))
        traffic = prof.get("dram_bytes_per_launch")
    except Exception:
        pass
    csum = clocks.summary()
    # the binding resource (ncu): the L1TEX data pipe, 1 wavefront / SM / cycle;
    # wavefronts per query from the committed capture, clock sampled live
    binding = None
    if prof.get("lsu_wavefronts_per_query") and csum.get("sm_mhz"):
        wpq = float(prof["lsu_wavefronts_per_query"])
        nsm = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
        ach = (n / (avg_launch_ms * 1e-3)) * wpq / (nsm * csum["sm_mhz"] * 1e6)
        pk = float(prof.get("lsu_wavefront_peak_per_sm_cycle", 1.0))
        binding = {"resource": "L1TEX data-pipe wavefronts (scattered hash-table gathers)",
                   "wavefronts_per_query": wpq, "achieved_per_sm_cycle": ach,
                   "peak_per_sm_cycle": pk, "frac": ach / pk,
                   "source": "profiles/full_forward_traffic.json (ncu) + live launch time "
                             "and SM clock"}
    # the measured random-gather peak of this pool's B200s (tools/l2_gather_peak.cu):
    # the hash-table slots levels 4-11 read from L2 per second against it
    l2peak = prof.get("l2_gather_peak") or {}
    l2_vs_peak = None
    if l2peak.get("slots_per_s_8B"):
        slots = n / (avg_launch_ms * 1e-3) * float(prof.get("l2_slots_per_query", 64))
        l2_vs_peak = {"slots_per_s": slots, "peak_slots_per_s_8B": l2peak["slots_per_s_8B"],
                      "frac": slots / l2peak["slots_per_s_8B"],
                      "note": "x-even corner pairs share one 16-byte load (2 slots), so the "
                              "kernel can exceed the 8-byte-gather peak; the paired-load peak "
                              "is " + f"{l2peak.get('pairs_per_s_16B', 0):.3g} loads/s",
                      "source": l2peak.get("source")}
    line = {
        "metric": "nirc_queries_per_sec", "value": value, "unit": "queries/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": cfg2_config(world),
        "kernel_precision": f"tcgen05 {'2xFP16-split' if PRECISION == 2 else '3xTF32'}",
        "roofline": {"bound": "hbm", "achieved": achieved_gbs, "peak": hbm_peak, "unit": "GB/s",
                     "frac": achieved_gbs / hbm_peak, "traffic": traffic,
                     "kernel": "k_full_forward_tc (+ k_pack_weights)",
                     "algorithmic_bytes_per_query": HBM_BYTES_PER_QUERY,
                     "avg_launch_ms": avg_launch_ms,
                     "tensor_tflops": tflops,
                     "tensor_frac": tflops / float(peaks.get("bf16_tflops", 1590.0)),
                     "l2_gather_gbs": l2_gbs,
                     "peak_source": "MEASURED_PEAKS.json" if peaks else "fallback",
                     "binding_resource": binding, "l2_gather_vs_measured_peak": l2_vs_peak},
        "clocks": csum,
        "e2e": {"value": e2e_value, "unit": "queries/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "steps": e2e_steps,
                "median_step_value": world * n / (e2e_per_step[len(e2e_per_step) // 2] * 1e-3),
                "step_ms_min_median_max": [round(e2e_per_step[0], 3),
                                           round(e2e_per_step[len(e2e_per_step) // 2], 3),
                                           round(e2e_per_step[-1], 3)],
                "variance_note": "value = all steps' mean; on some boxes single steps (and "
                                 "rarely whole windows) of the host copies run slower, so "
                                 "the per-step median is given beside it",
                "path": "paper_2412_04634_b200.mlp.full_forward on pinned host tensors (chunked "
                        "H2D / fused kernel / D2H pipeline inside the call)",
                "numpy_caller": e2e_numpy, "pcie_roofline": e2e_pcie},
        "gpu_launches": 2 * args.steps,
    }
    if fb is not None:
        line["frame_1080p"] = fb
        seq = fb.get("sequential", fb)
        line["frame_1080p_ms"] = fb["value"]
        line["train_samples_per_sec"] = seq.get("train_samples_per_sec")
        line["infer_roofline"] = seq.get("infer_roofline")
        if "cfg5_4k" in fb:
            line["frame_4k_ms"] = fb["cfg5_4k"]["value"]
        if "cfg1_128" in fb:
            line["frame_128_ms"] = fb["cfg1_128"]["value"]
    if world == 1 and not args.no_cpu_baseline:
        # ~10 s of single-core work: 64 chunks of 2^15 random cfg2 queries
        rate, nq = cpu_baseline(cores=1, chunks=64, chunk=1 << 15)
        line["cpu_baseline"] = {"value": rate, "unit": "queries/s", "cores": 1, "kind": "port",
                                "sample": f"{nq} random cfg2 queries (64 chunks of 2^15) through "
                                          "oracle/nirc_oracle.full_forward (numpy "
                                          "encode_batch + mlp_forward, OPENBLAS 1 thread)",
                                "host": host_info()}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_rank % torch.cuda.device_count())
        # NCCL over NVLink; NIRC_DIST_BACKEND=gloo lets several ranks share
        # one GPU (a smoke test of the multi-rank path on a 1-GPU box)
        dist.init_process_group(os.environ.get("NIRC_DIST_BACKEND", "nccl"))
    run_b200(args, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
