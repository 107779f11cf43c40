"""Benchmark: ms per reference-to-all-vertex NDF query (250x352x20 = 1.76 M vertices).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one full reference-to-all-vertices NDF query (BASELINE config 1):
fused embed + [e_r+e_q, |e_r-e_q|] + 4x128 SiLU MLP (tcgen05, fp32 TMEM
accumulation) + tanh head over all vertices.  With N > 1 ranks (torchrun, one
GPU per rank, NCCL) the vertex range is split into N contiguous shards
(strong scaling: total work fixed) and the field is assembled with one NCCL
all-gather inside the timed step.  Inputs (model, latent grid) are resident in
HBM; the L2 (126 MB) is flushed with a 512 MB write between timed steps since
the query's working set would otherwise stay cached.  Device time is measured
with CUDA events on the launching stream; the reported value is the max over
ranks.

Secondary lines in the same JSON object: the ground-truth Pearson GEMV over the
z-scored 1000 x 1.76 M ensemble (HBM roofline), the KSG-MI field throughput on
config 2 (pairs/s), and the host-CPU reference timed on this box.

``--impl reference`` times the reference's CPU implementation of the query
(the oracle restatement, oracle/ndf_oracle.py -- the reference is pure Python
and cannot be installed on the GPU box) with all host cores on a bounded
seeded vertex sample per step, extrapolated to the full grid.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ms per ref-to-all-vertex NDF query (1.76M vtx)"
PAPER_MS = 9.0          # PAPER.md:344/350, RTX 3090
FLOP_PER_PAIR = 2 * (110 * 128 + 128 * 128 * 2 + 128)   # 93,952


def load_traffic():
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as fh:
            return json.load(fh)
    except (OSError, ValueError):
        return {}


SFU_OPS_PER_PAIR = 3 * 128      # one tanh.approx per hidden activation
SFU_PER_CLK_SM = 16             # measured, tools/micro/mufu_rate.cu


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)

class ClockSampler:
    """SM clock + throttle reasons sampled DURING the timed region.

    NVML polled from a thread every ~0.5 ms (the timed region of a default run is only
    tens of ms), falling back to ``nvidia-smi -lms 50``.  One sample is taken before
    the region starts and one after it ends, so the region is bracketed."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index=0, interval_s=0.0005):
        self.index = index
        self.interval = interval_s
        self.samples = []          # (sm_mhz, max_mhz, set of reasons)
        self.proc = None
        self.nvml = None
        self._run = False

    def _nvml_sample(self):
        n = self.nvml
        sm = n.nvmlDeviceGetClockInfo(self.handle, n.NVML_CLOCK_SM)
        mask = n.nvmlDeviceGetCurrentClocksEventReasons(self.handle)
        bits = {"hw_slowdown": getattr(n, "nvmlClocksEventReasonHwSlowdown", 0x8),
                "hw_thermal_slowdown": getattr(n, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
                "sw_thermal_slowdown": getattr(n, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
                "sw_power_cap": getattr(n, "nvmlClocksEventReasonSwPowerCap", 0x4)}
        self.samples.append((float(sm), float(self.max_sm),
                             {k for k, b in bits.items() if mask & b}))

    def _nvml_loop(self):
        while self._run:
            try:
                self._nvml_sample()
            except Exception:
                return
            time.sleep(self.interval)

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.handle = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_sm = pynvml.nvmlDeviceGetMaxClockInfo(self.handle, pynvml.NVML_CLOCK_SM)
            self._nvml_sample()
            self._run = True
            self.thread = threading.Thread(target=self._nvml_loop, daemon=True)
            self.thread.start()
            return self
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            t0 = time.time()
            while not self.samples and time.time() - t0 < 10 and self.proc.poll() is None:
                time.sleep(0.01)
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 6 and parts[0].replace(".", "").isdigit():
                reasons = {self.NAMES[i] for i in range(4) if parts[2 + i].lower() == "active"}
                mx = float(parts[1]) if parts[1].replace(".", "").isdigit() else 0.0
                self.samples.append((float(parts[0]), mx, reasons))

    def __exit__(self, *exc):
        if self.nvml is not None:
            self._run = False
            self.thread.join(timeout=2)
            try:
                self._nvml_sample()           # one sample after the region
            except Exception:
                pass
            return
        n = len(self.samples)
        t0 = time.time()
        while self.proc is not None and len(self.samples) <= n and time.time() - t0 < 2:
            time.sleep(0.01)
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [s[0] for s in self.samples]
        return {"sm_mhz": statistics.median(sm), "sm_min_mhz": min(sm),
                "sm_max_mhz": max(s[1] for s in self.samples),
                "reasons": sorted(set().union(*(s[2] for s in self.samples))),
                "samples": len(self.samples),
                "source": "nvml 0.5 ms" if self.nvml is not None else "nvidia-smi 50 ms"}


# ---------------------------------------------------------------------------
# distributed plumbing

def dist_setup(n_gpus):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------------------
# CPU reference (oracle) timing -- rank 0 only


_WORKER_MODEL = None


def _oracle_init(model_arrays, ref, dims):
    """Pool initializer: the model is shipped to each worker once, not per task."""
    global _WORKER_MODEL
    from oracle import ndf_oracle as O
    _WORKER_MODEL = (O.OracleModel(*model_arrays), ref, dims)


def _oracle_chunk(idx):
    from oracle import ndf_oracle as O
    om, ref, dims = _WORKER_MODEL
    return O.reconstruct_field(om, ref, dims, vertices=idx)


def oracle_pool(model, w, procs):
    from concurrent.futures import ProcessPoolExecutor
    arrays = (model.spec.fourier_octaves, model.grid_mu, model.grid_nu, model.weights,
              model.biases, model.spec.merge, model.spec.activation, model.spec.head_kind)
    return ProcessPoolExecutor(max_workers=procs, initializer=_oracle_init,
                               initargs=(arrays, w.ref_position(), w.dims))


def cpu_query_rate(model, w, sample, procs, pool=None, seed=1):
    """Seconds per vertex of the reference-restated query over a seeded sample
    (wall time of `procs` worker processes, model already resident in the workers)."""
    idx = np.random.default_rng(seed).choice(w.n_vertices, size=sample, replace=False)
    chunks = np.array_split(idx, procs)
    own = pool is None
    pool = pool or oracle_pool(model, w, procs)
    try:
        list(pool.map(_oracle_chunk, [c[:8] for c in chunks]))
        t0 = time.perf_counter()     # pool warm; time the sample only
        list(pool.map(_oracle_chunk, chunks))
        dt = time.perf_counter() - t0
    finally:
        if own:
            pool.shutdown()
    return dt / sample, dt


def _ksg_chunk(args):
    from oracle import ndf_oracle as O
    ref_vec, cols, k = args
    return [O.ksg_mi(ref_vec, c, k) for c in cols]


def cpu_ksg_rate(X, ref_flat, idx, k, procs):
    from concurrent.futures import ProcessPoolExecutor
    ref_vec = X[:, ref_flat].astype(np.float64)
    cols = [X[:, v].astype(np.float64) for v in idx]
    parts = [cols[i::procs * 2] for i in range(procs * 2)]
    t0 = time.perf_counter()
    with ProcessPoolExecutor(max_workers=procs) as ex:
        list(ex.map(_ksg_chunk, [(ref_vec, p, k) for p in parts]))
    dt = time.perf_counter() - t0
    return len(idx) / dt, dt


# ---------------------------------------------------------------------------


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2307_02203_b200 import workloads as W
    w = W.CONFIGS[1]
    model = W.build_model(w, seed=0, grid_init=1e-4)
    procs = os.cpu_count() or 1
    sample = args.ref_sample
    times = []
    with oracle_pool(model, w, procs) as pool:
        for i in range(args.warmup + args.steps):
            per_vertex, _ = cpu_query_rate(model, w, sample, procs, pool=pool, seed=1 + i)
            if i >= args.warmup:
                times.append(per_vertex * w.n_vertices * 1e3)
    ms = statistics.mean(times)
    line = {
        "impl": "reference", "metric": METRIC, "value": ms, "unit": "ms",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": False, "scaling": "strong", "vs_baseline": ms / PAPER_MS,
        "dtype": "f32", "data": "synthetic",
        "config": {"workload": w.name, "vertices": w.n_vertices, "mlp": [110, 128, 128, 128, 1],
                   "parallelism": "host processes"},
        "cpu_baseline": {"value": ms, "unit": "ms", "cores": procs, "kind": "port",
                         "sample": f"{sample} seeded vertices per step via oracle/ndf_oracle.py "
                                   f"reconstruct_field (einsum exact, reference order), "
                                   f"extrapolated x{w.n_vertices / sample:.1f}"},
        "e2e": {"value": ms, "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch
    import paper_2307_02203_b200 as ndf
    from paper_2307_02203_b200 import _native as N
    from paper_2307_02203_b200 import workloads as W

    rank, world, local = dist_setup(args.gpus)
    dev = torch.device("cuda", torch.cuda.current_device())
    peaks, peak_kind = load_peaks()
    w = W.CONFIGS[1]
    V = w.n_vertices
    shard = math.ceil(V / world)
    v0, v1 = min(V, rank * shard), min(V, (rank + 1) * shard)
    model = W.build_model(w, seed=0, grid_init=1e-4).with_precision(args.precision)
    st = model.device_state(dev)
    ref = w.ref_position()
    local_out = torch.empty(shard, dtype=torch.float32, device=dev)
    full = torch.empty(shard * world, dtype=torch.float32, device=dev) if world > 1 else None
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        ndf.reconstruct_field_device(model, ref, ndf.ROLE_MU, w.dims, v0, v1,
                                     out=local_out[: v1 - v0])
        if world > 1:
            import torch.distributed as dist
            dist.all_gather_into_tensor(full, local_out)

    for _ in range(args.warmup):
        flush.fill_(1.0)
        step()
    torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    N.launch_count(reset=True)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    kstarts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    kends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.fill_(float(i))
            starts[i].record(stream)
            kstarts[i].record(stream)
            ndf.reconstruct_field_device(model, ref, ndf.ROLE_MU, w.dims, v0, v1,
                                         out=local_out[: v1 - v0])
            kends[i].record(stream)
            if world > 1:
                import torch.distributed as dist
                dist.all_gather_into_tensor(full, local_out)
            ends[i].record(stream)
        torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    launches = N.launch_count(reset=True)
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    kern_ms = [s.elapsed_time(e) for s, e in zip(kstarts, kends)]
    ms = max_over_ranks(statistics.mean(step_ms), world)
    kms = max_over_ranks(statistics.mean(kern_ms), world)
    clocks = clk.summary()

    # e2e through the public API: host result, pinned D2H inside the timed region
    e2e_ms = None
    if rank == 0:
        ts = []
        for i in range(args.warmup + args.steps):
            flush.fill_(float(i))
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            grid = ndf.reconstruct_field(model, ref, ndf.ROLE_MU, w.dims)
            ts.append((time.perf_counter() - t0) * 1e3)
            del grid
        e2e_ms = statistics.mean(ts[args.warmup:])

    line = None
    if rank == 0:
        achieved_tflops = FLOP_PER_PAIR * (v1 - v0) / (kms * 1e-3) / 1e12
        peak = peaks.get("bf16_tflops", 1590.0)
        traffic = load_traffic()
        sm_count = torch.cuda.get_device_properties(dev).multi_processor_count
        sm_hz = (clocks.get("sm_mhz") or peaks.get("sm_max_mhz", 1965.0)) * 1e6
        sfu_floor_ms = SFU_OPS_PER_PAIR * (v1 - v0) / (SFU_PER_CLK_SM * sm_count * sm_hz) * 1e3
        line = {
            "metric": METRIC, "value": ms, "unit": "ms", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": ms / PAPER_MS,
            "dtype": args.precision, "data": "synthetic",
            "config": {"workload": w.name, "vertices": V, "grid": list(w.dims),
                       "latent": list(model.spec.latent_resolution) + [16],
                       "mlp": model.spec.decoder_widths(), "head": model.spec.head_kind,
                       "parallelism": f"vertex-shard x{world} + NCCL all-gather",
                       "sms": sm_count,
                       "l2": "flushed (512 MB write) between timed steps"},
            "roofline": {"bound": "tensor", "kernel": "ndf::tc::query_pp_kernel (+ prep_ws_feat_kernel, prep_ws_merge_kernel)",
                         "achieved": achieved_tflops, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved_tflops / peak, "peak_kind": f"{peak_kind} bf16 burst",
                         "kernel_ms": kms, "flop_per_launch": FLOP_PER_PAIR * (v1 - v0),
                         "traffic": traffic.get("query_pp_kernel"),
                         "sfu_floor_ms": sfu_floor_ms, "sfu_frac": sfu_floor_ms / kms},
            "clocks": clocks,
            "gpu_launches": launches,
            "e2e": {"value": e2e_ms, "unit": "ms", "h2d_bytes_per_step": 24,
                    "d2h_bytes_per_step": 4 * V,
                    "api": "paper_2307_02203_b200.reconstruct_field -> FieldGrid (host)",
                    "d2h": "kernel stores into pinned host memory (zero-copy)",
                    "scope": "one GPU (rank 0): the public call is single-device"
                             if world > 1 else "one GPU"},
        }
    if not args.quick:
        secondary(args, line, rank, world, dev, peaks, peak_kind, model, w)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def secondary(args, line, rank, world, dev, peaks, peak_kind, model, w):
    """Pearson GEMV (c1), KSG field throughput (c2), CPU baseline (rank 0, N=1)."""
    import torch
    import paper_2307_02203_b200 as ndf
    from paper_2307_02203_b200 import _native as N
    from paper_2307_02203_b200 import workloads as W
    stream = torch.cuda.current_stream(dev)
    V = w.n_vertices
    shard = math.ceil(V / world)
    v0, v1 = min(V, rank * shard), min(V, (rank + 1) * shard)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    # ---- Pearson GEMV over Z ---------------------------------------------------
    ens = W.generate_device(w, dev)
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    pz0 = torch.cuda.Event(enable_timing=True)
    pz1 = torch.cuda.Event(enable_timing=True)
    pz0.record(stream)
    Z, norm = ens.zscore()
    pz1.record(stream)
    torch.cuda.synchronize()
    zscore_ms = pz0.elapsed_time(pz1)
    M = ens.member_count
    ref_flat = w.ref_flat()
    zref = Z[:, ref_flat].contiguous()
    out = torch.empty(v1 - v0, dtype=torch.float32, device=dev)
    g_ms = []
    for i in range(args.warmup + args.steps):
        flush.fill_(float(i))
        t0.record(stream)
        N.call("ndf_pearson_gemv", N.ptr(Z), N.ptr(norm), M, V, N.ptr(zref), 0, v0, v1, N.ptr(out),
               N.stream_handle(dev))
        t1.record(stream)
        torch.cuda.synchronize()
        if i >= args.warmup:
            g_ms.append(t0.elapsed_time(t1))
    gms = max_over_ranks(statistics.mean(g_ms), world)
    gbytes = 4.0 * M * (v1 - v0) + 4.0 * (v1 - v0) * 2
    hbm = peaks.get("hbm_gbs", 6650.0)
    gemv_gbs = gbytes / (gms * 1e-3) / 1e9
    # ---- KSG field on config 2 --------------------------------------------------
    del Z, norm, zref
    ens.drop_derived()
    del ens
    torch.cuda.empty_cache()
    w2 = W.CONFIGS[2]
    ens2 = W.generate_device(w2, dev)
    ksg_n = args.ksg_pairs
    k_v0 = v0
    k_v1 = min(v1, v0 + ksg_n)
    ref_vec = ens2.X.reshape(ens2.member_count, -1)[:, w2.ref_flat()].double().contiguous()
    from paper_2307_02203_b200.measures import _KsgTables
    jit, psi = _KsgTables.get(dev, ens2.member_count)
    mi = torch.empty(k_v1 - k_v0, dtype=torch.float32, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    psi_km = _KsgTables.psi_km(w2.ksg_k, ens2.member_count)
    k_ms = []
    for i in range(1 + max(1, args.steps // 5)):
        t0.record(stream)
        N.call("ndf_ksg_ref_nodes", N.ptr(ens2.X), ens2.member_count, V, N.ptr(ref_vec), k_v0, k_v1,
               w2.ksg_k, N.ptr(jit), N.ptr(psi), psi_km, None, N.ptr(mi), None, N.ptr(status),
               N.stream_handle(dev))
        t1.record(stream)
        torch.cuda.synchronize()
        if i >= 1:
            k_ms.append(t0.elapsed_time(t1))
    kms = statistics.mean(k_ms)
    pairs_s = (k_v1 - k_v0) / (kms * 1e-3) * world
    if rank == 0:
        line["pearson_gemv"] = {
            "ms": gms, "bytes": gbytes, "achieved_gbs": gemv_gbs, "peak_gbs": hbm,
            "frac": gemv_gbs / hbm, "peak_kind": f"{peak_kind} hbm copy",
            "traffic": load_traffic().get("gemv_kernel"),
            "zscore_prep_ms": zscore_ms, "members": M, "vertices": v1 - v0}
        line["ksg_mi"] = {"pairs_per_s": pairs_s, "unit": "pairs/s", "k": w2.ksg_k,
                          "members": ens2.member_count, "sample_pairs": k_v1 - k_v0,
                          "ms": kms, "full_field_s_extrapolated": V / pairs_s}
    # ---- config 4: bulk estimator pairs (Pearson + KSG), sharded pair ranges ---------
    n_pairs = args.c4_pairs
    pa_all, pb_all = W.pair_list(W.CONFIGS[4], count=n_pairs, seed=2)
    p0, p1 = min(n_pairs, rank * math.ceil(n_pairs / world)), min(n_pairs, (rank + 1) * math.ceil(n_pairs / world))
    ens2.vertex_major()
    # warm-up on a slice (kernel attributes, psi / jitter tables, allocator), then time
    ndf.pair_estimators_device(ens2, "v", pa_all[p0:p0 + 1024], pb_all[p0:p0 + 1024],
                               k=W.CONFIGS[4].ksg_k)
    torch.cuda.synchronize()
    t0.record(stream)
    res = ndf.pair_estimators_device(ens2, "v", pa_all[p0:p1], pb_all[p0:p1], k=W.CONFIGS[4].ksg_k)
    t1.record(stream)
    torch.cuda.synchronize()
    c4_ms = max_over_ranks(t0.elapsed_time(t1), world)
    del res
    ens2.drop_derived()
    if rank == 0:
        line["c4_bulk_pairs"] = {"pairs": n_pairs, "ms": c4_ms, "pairs_per_s": n_pairs / (c4_ms * 1e-3),
                                 "estimators": ["pearson", "ksg_mi"], "k": W.CONFIGS[4].ksg_k,
                                 "note": "seeded pair list (half uniform, half within +-16 cells), "
                                         "subset of the 2^22 config-4 list; vertex-major copy built "
                                         "before timing"}
    # ---- config 3: 64-reference fp16 cube, both heads ---------------------------------
    w3 = W.CONFIGS[3]
    refs = W.reference_vertices(w3, count=64, seed=1)
    pos = np.stack([np.array([2.0 * i / (n - 1) - 1.0 for i, n in
                              zip((v % w3.dims[0], (v // w3.dims[0]) % w3.dims[1],
                                   v // (w3.dims[0] * w3.dims[1])), w3.dims)]) for v in refs])
    models = [W.build_model(w3, seed=0, grid_init=1e-4).with_precision(args.precision),
              ndf.NdfModel.build(
                  ndf.ModelSpec.baseline(w3.dims, w3.latent_factor, measure_kind="ksg_mi",
                                         precision=args.precision), seed=1)]
    cube = torch.empty((64, v1 - v0), dtype=torch.float16, device=dev)
    c3 = []
    for i in range(1 + max(1, args.steps // 5)):
        torch.cuda.synchronize()
        t0.record(stream)
        for m3 in models:
            ndf.reconstruct_multi_device(m3, pos, ndf.ROLE_MU, w3.dims, v0, v1, out=cube)
        t1.record(stream)
        torch.cuda.synchronize()
        if i:
            c3.append(t0.elapsed_time(t1))
    c3_ms = max_over_ranks(statistics.mean(c3), world)
    if rank == 0:
        line["c3_multi_ref"] = {"refs": 64, "heads": 2, "pairs": 2 * 64 * V, "ms": c3_ms,
                                "pairs_per_s": 2 * 64 * V / (c3_ms * 1e-3),
                                "tflops": FLOP_PER_PAIR * 2 * 64 * V / (c3_ms * 1e-3) / 1e12,
                                "output": "fp16 cube 64 x 1.76M per head"}
    del cube
    # ---- the reference's own default architecture (HashGrid + encoder
    # MLPs, exact fp32 path) queried over the config-1 grid ------------------------------
    mref = ndf.NdfModel.build(ndf.ModelSpec.reference_default(), seed=0)
    outr = torch.empty(v1 - v0, dtype=torch.float32, device=dev)
    f3 = []
    for i in range(1 + max(1, args.steps // 5)):
        flush.fill_(float(i))
        t0.record(stream)
        ndf.reconstruct_field_device(mref, w.ref_position(), ndf.ROLE_MU, w.dims, v0, v1, out=outr)
        t1.record(stream)
        torch.cuda.synchronize()
        if i:
            f3.append(t0.elapsed_time(t1))
    f3_ms = max_over_ranks(statistics.mean(f3), world)
    if rank == 0:
        spec = mref.spec
        line["f3_reference_default"] = {
            "ms": f3_ms, "vertices": V, "precision": "fp32 (exact, matmul_exact order)",
            "model": f"reference ModelSpec(): {spec.levels}-level HashGrid 2^{spec.log2_table_size}"
                     f"x{spec.features_per_level}, encoders {spec.encoder_widths()}, decoder "
                     f"{spec.decoder_widths()}, {spec.merge} merge, snake_alt, linear head"}
    del outr, mref
    # ---- CPU baseline (rank 0, N=1 only) -----------------------------------------
    if rank == 0 and world == 1 and not args.no_cpu:
        procs = os.cpu_count() or 1
        per_v, dt = cpu_query_rate(model.with_precision("fp32"), w, args.cpu_sample, procs)
        cpu_ms = per_v * V * 1e3
        line["cpu_baseline"] = {
            "value": cpu_ms, "unit": "ms", "cores": procs, "kind": "port",
            "sample": f"{args.cpu_sample} seeded vertices of config 1 via oracle/ndf_oracle.py "
                      f"reconstruct_field (reference einsum order) in {procs} processes, "
                      f"{dt:.1f} s wall, extrapolated to {V} vertices"}
        X2 = ens2.X.reshape(ens2.member_count, -1)
        idx = np.random.default_rng(3).choice(V, size=args.cpu_ksg_pairs, replace=False)
        Xh = X2[:, torch.from_numpy(np.append(idx, w2.ref_flat())).to(dev)].cpu().numpy()
        rate, kdt = cpu_ksg_rate(Xh, Xh.shape[1] - 1, np.arange(len(idx)), w2.ksg_k, procs)
        line["ksg_mi"]["cpu_pairs_per_s"] = rate
        line["ksg_mi"]["cpu_sample"] = (f"{len(idx)} seeded config-2 vertices, oracle ksg_mi "
                                        f"(scipy cKDTree, reference algorithm) in {procs} "
                                        f"processes, {kdt:.1f} s wall")
        line["ksg_mi"]["speedup_vs_cpu"] = pairs_s / rate


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--precision", choices=["fp16", "bf16", "fp32"], default="fp16")
    ap.add_argument("--quick", action="store_true", help="query only (profiling runs)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=1 << 19)
    ap.add_argument("--cpu-ksg-pairs", type=int, default=2048)
    ap.add_argument("--ksg-pairs", type=int, default=1 << 15)
    ap.add_argument("--ref-sample", type=int, default=1 << 18)
    ap.add_argument("--c4-pairs", type=int, default=1 << 16)
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
