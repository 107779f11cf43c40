"""Benchmark: ms per reference-to-all-vertex NDF query (250x352x20 = 1.76 M vertices).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one full reference-to-all-vertices NDF query (BASELINE config 1):
fused embed + [e_r+e_q, |e_r-e_q|] + 4x128 SiLU MLP (tcgen05, bf16 operands,
fp32 TMEM accumulation) + tanh head over all vertices.  With N > 1 ranks (torchrun, one
GPU per rank, NCCL) the vertex range is split into N contiguous shards
(strong scaling: total work fixed) and the field is assembled with one NCCL
all-gather inside the timed step.  Inputs (model, latent grid) are resident in
HBM; the L2 (126 MB) is flushed with a 512 MB write between timed steps since
the query's working set would otherwise stay cached.  Device time is measured
with CUDA events on the launching stream; the reported value is the max over
ranks.

The headline runs the config's own dtype, bf16 (split hi/lo operands on
tcgen05, fp32 TMEM accumulation, max|err| vs the fp32 oracle reported in
"parity"); fp16 is timed the same way as a secondary key.

Secondary lines in the same JSON object: config 0 (GPU and CPU), the ground-
truth Pearson GEMV over the z-scored 1000 x 1.76 M ensemble (HBM roofline) and
the fresh-ensemble path, the KSG-MI field on config 2 (full field, plus the
CPU's own vertex sample timed on both sides), the full 2^22-pair config-4 list,
the 64-reference cube of config 3, and the host-CPU reference on this box.

``--impl reference`` times the reference's CPU implementation of the query
(the oracle restatement, oracle/ndf_oracle.py -- the reference is pure Python
and cannot be installed on the GPU box) with all host cores, the full grid per
step.
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


def cpu_sample_size(model, w, procs, pool, want, step_s):
    """Vertices per CPU step: the full grid (``want``) unless this host's measured rate
    would make a step longer than ``step_s`` seconds -- then the largest seeded sample
    that fits (reported as extrapolated), so a run stays within minutes on slow hosts."""
    want = min(want, w.n_vertices)
    probe = min(want, 65536)
    per_v, _ = cpu_query_rate(model, w, probe, procs, pool=pool, seed=999)
    if per_v * want <= step_s:
        return want
    return max(probe, min(want, int(step_s / per_v)))


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
    """The reference arm: the reference's CPU query path (oracle port of reconstruct_field,
    reference einsum order) on all host cores.  Each step is the FULL config-1 grid
    (1.76 M vertices) -- measured, not extrapolated."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2307_02203_b200 import workloads as W
    w = W.CONFIGS[1]
    model = W.build_model(w, seed=0, grid_init=1e-4)
    procs = os.cpu_count() or 1
    times = []
    with oracle_pool(model, w, procs) as pool:
        sample = cpu_sample_size(model, w, procs, pool, args.ref_sample, args.ref_step_s)
        for i in range(args.warmup + args.steps):
            per_vertex, _ = cpu_query_rate(model, w, sample, procs, pool=pool, seed=1 + i)
            if i >= args.warmup:
                times.append(per_vertex * w.n_vertices * 1e3)
    ms = statistics.mean(times)
    scope = ("the full grid per step (no extrapolation)" if sample == w.n_vertices else
             f"{sample} seeded vertices per step, extrapolated x{w.n_vertices / sample:.2f}")
    line = {
        "impl": "reference", "metric": METRIC, "value": ms, "unit": "ms",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": False, "scaling": "strong", "vs_baseline": ms / PAPER_MS,
        "dtype": "f32", "data": "synthetic",
        "config": {"workload": w.name, "vertices": w.n_vertices, "mlp": [110, 128, 128, 128, 1],
                   "parallelism": "host processes"},
        "cpu_baseline": {"value": ms, "unit": "ms", "cores": procs, "kind": "port",
                         "sample": f"oracle/ndf_oracle.py reconstruct_field (einsum exact, "
                                   f"reference order) over {scope}; step times min/max "
                                   f"{min(times):.0f}/{max(times):.0f} ms"},
        "e2e": {"value": ms, "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# x3 (bf16 split operands) issues per 128-row tile: layer 0 = 3 selector + 6 latent K16
# MMAs, each hidden layer = bias + 3 x 8 K16 MMAs (A_hi W_hi, A_lo W_hi, A_hi W_lo);
# tiles are 16 x 8 nodes (ceil(250/16) x ceil(7040/8) tiles at config 1)
X3_MMAS_PER_TILE = 9 + 2 * 25
MMA_FLOP = 2 * 128 * 128 * 16


def issued_tensor_flop(precision, dims):
    nx, ny, nz = dims
    if precision == "bf16":
        tiles = math.ceil(nx / 16) * math.ceil(ny * nz / 8)
        return tiles * X3_MMAS_PER_TILE * MMA_FLOP
    tiles = math.ceil(nx * ny * nz / 128)
    return tiles * (8 + 2 * 9) * MMA_FLOP          # fp16 ping-pong: bias + 7, bias + 8 (x2)


def time_query(model, w, v0, v1, steps, warmup, world, dev, flush, clocks=True):
    """Per-step device time (CUDA events on the launching stream, L2 flushed between
    steps), the query-only time, launches and the clock record."""
    import torch
    import paper_2307_02203_b200 as ndf
    from paper_2307_02203_b200 import _native as N
    stream = torch.cuda.current_stream(dev)
    shard = v1 - v0 if world == 1 else math.ceil(w.n_vertices / world)
    local_out = torch.empty(shard, dtype=torch.float32, device=dev)
    full = torch.empty(shard * world, dtype=torch.float32, device=dev) if world > 1 else None
    ref = w.ref_position()

    def step():
        ndf.reconstruct_field_device(model, ref, ndf.ROLE_MU, w.dims, v0, v1,
                                     out=local_out[: v1 - v0])

    for _ in range(warmup):
        flush.fill_(1.0)
        step()
        if world > 1:
            import torch.distributed as dist
            dist.all_gather_into_tensor(full, local_out)
    torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    N.launch_count(reset=True)
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(steps)] for _ in range(3)]
    with (ClockSampler(int(os.environ.get("LOCAL_RANK", "0"))) if clocks else _NoClock()) as clk:
        for i in range(steps):
            flush.fill_(float(i))
            ev[0][i].record(stream)
            step()
            ev[1][i].record(stream)
            if world > 1:
                import torch.distributed as dist
                dist.all_gather_into_tensor(full, local_out)
            ev[2][i].record(stream)
        torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    launches = N.launch_count(reset=True)
    step_ms = max_over_ranks(statistics.mean(a.elapsed_time(b) for a, b in zip(ev[0], ev[2])), world)
    kern_ms = max_over_ranks(statistics.mean(a.elapsed_time(b) for a, b in zip(ev[0], ev[1])), world)
    return step_ms, kern_ms, launches, clk.summary()


class _NoClock:
    def __enter__(self):
        return self

    def __exit__(self, *exc):
        return False

    def summary(self):
        return None


def run_ours(args):
    import torch
    import paper_2307_02203_b200 as ndf
    from paper_2307_02203_b200 import workloads as W

    rank, world, local = dist_setup(args.gpus)
    dev = torch.device("cuda", torch.cuda.current_device())
    peaks, peak_kind = load_peaks()
    w = W.CONFIGS[1]
    V = w.n_vertices
    shard = math.ceil(V / world)
    v0, v1 = min(V, rank * shard), min(V, (rank + 1) * shard)
    base = W.build_model(w, seed=0, grid_init=1e-4)
    model = base.with_precision(args.precision)
    model.device_state(dev)
    ref = w.ref_position()
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    ms, kms, launches, clocks = time_query(model, w, v0, v1, args.steps, args.warmup, world, dev,
                                           flush)
    # the other 16-bit precision, same protocol (secondary key)
    alt = "fp16" if args.precision == "bf16" else "bf16"
    alt_ms = alt_kms = None
    if args.precision != "fp32":
        alt_ms, alt_kms, _, _ = time_query(base.with_precision(alt), w, v0, v1, args.steps,
                                           args.warmup, world, dev, flush, clocks=False)

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
        flop = FLOP_PER_PAIR * (v1 - v0)
        achieved_tflops = flop / (kms * 1e-3) / 1e12
        peak = peaks.get("bf16_tflops", 1590.0)
        traffic = load_traffic()
        sm_count = torch.cuda.get_device_properties(dev).multi_processor_count
        sm_hz = ((clocks or {}).get("sm_mhz") or peaks.get("sm_max_mhz", 1965.0)) * 1e6
        sfu_floor_ms = SFU_OPS_PER_PAIR * (v1 - v0) / (SFU_PER_CLK_SM * sm_count * sm_hz) * 1e3
        kname = {"bf16": "ndf::tc::query_x3_kernel (+ prep_x3_kernel)",
                 "fp16": "ndf::tc::query_pp_kernel (+ prep_ws_feat_kernel, prep_ws_merge_kernel)",
                 "fp32": "ndf::query_f32_kernel (+ prep)"}[args.precision]
        roof = {"bound": "tensor", "kernel": kname,
                "achieved": achieved_tflops, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved_tflops / peak, "peak_kind": f"{peak_kind} bf16 burst",
                "kernel_ms": kms, "flop_per_launch": flop,
                "flop_basis": f"algorithmic {FLOP_PER_PAIR} FLOP per pair (SURVEY 8(d))",
                "traffic": traffic.get({"bf16": "query_x3_kernel"}.get(args.precision,
                                                                        "query_pp_kernel")),
                "sfu_floor_ms": sfu_floor_ms, "sfu_frac": sfu_floor_ms / kms}
        if args.precision != "fp32" and world == 1:
            issued = issued_tensor_flop(args.precision, w.dims)
            roof["issued_tensor_flop_per_launch"] = issued
            roof["issued_tflops"] = issued / (kms * 1e-3) / 1e12
            roof["issued_frac"] = roof["issued_tflops"] / peak
            if args.precision == "bf16":
                roof["issued_note"] = ("split operands: each hidden K16 step runs A_hi W_hi + "
                                       "A_lo W_hi + A_hi W_lo; layer 0 is 3 selector + 6 latent "
                                       "MMAs; 16x8-node tiles")
        line = {
            "metric": METRIC, "value": ms, "unit": "ms", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": ms / PAPER_MS,
            "dtype": args.precision, "data": "synthetic",
            "config": {"workload": w.name, "vertices": V, "grid": list(w.dims),
                       "latent": list(model.spec.latent_resolution) + [16],
                       "mlp": model.spec.decoder_widths(), "head": model.spec.head_kind,
                       "mlp_precision": {"bf16": "bf16 tcgen05 MMAs on split hi/lo operands, "
                                                 "fp32 TMEM accumulation",
                                         "fp16": "fp16 tcgen05 MMAs, fp32 TMEM accumulation",
                                         "fp32": "fp32 SIMT, reference summation order"}[
                           args.precision],
                       "parallelism": f"vertex-shard x{world} + NCCL all-gather",
                       "sms": torch.cuda.get_device_properties(dev).multi_processor_count,
                       "l2": "flushed (512 MB write) between timed steps"},
            "roofline": roof,
            "clocks": clocks,
            "gpu_launches": launches,
            "e2e": {"value": e2e_ms, "unit": "ms", "h2d_bytes_per_step": 24,
                    "d2h_bytes_per_step": 4 * V,
                    "api": "paper_2307_02203_b200.reconstruct_field -> FieldGrid (host)",
                    "d2h": "kernel stores into pinned host memory (zero-copy)",
                    "scope": "one GPU (rank 0): the public call is single-device"
                             if world > 1 else "one GPU"},
        }
        if alt_ms is not None:
            line[alt] = {"ms": alt_ms, "kernel_ms": alt_kms,
                         "tflops": FLOP_PER_PAIR * (v1 - v0) / (alt_kms * 1e-3) / 1e12,
                         "frac": FLOP_PER_PAIR * (v1 - v0) / (alt_kms * 1e-3) / 1e12 / peak}
        line["parity"] = parity_line(base, w, dev)
    if not args.quick:
        secondary(args, line, rank, world, dev, peaks, peak_kind, model, w)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def parity_line(base, w, dev, n=4096):
    """max|err| of each precision vs the oracle (fp32 reference restatement) on a seeded
    vertex subset of the benched model -- the number the timed kernels are held to."""
    import paper_2307_02203_b200 as ndf
    from oracle import ndf_oracle as O
    idx = np.sort(np.random.default_rng(11).choice(w.n_vertices, n, replace=False))
    om = O.OracleModel(base.spec.fourier_octaves, base.grid_mu, base.grid_nu, base.weights,
                       base.biases, base.spec.merge, base.spec.activation, base.spec.head_kind)
    want = O.reconstruct_field(om, w.ref_position(), w.dims, vertices=idx)
    out = {"vertices": n, "oracle": "oracle/ndf_oracle.py reconstruct_field",
           "tolerance": {"fp32": 1e-5, "bf16": 1e-2, "fp16": 1e-2}}
    for prec in ("bf16", "fp16", "fp32"):
        got = ndf.reconstruct_field_device(base.with_precision(prec), w.ref_position(),
                                           ndf.ROLE_MU, w.dims).cpu().numpy()
        out[f"max_abs_err_{prec}"] = float(np.max(np.abs(got[idx] - want)))
    return out


def _c4_cpu_chunk(args):
    from oracle import ndf_oracle as O
    A, B, k = args
    return [(float(O.pearson_rowwise(a[None], b[None])[0]), O.ksg_mi(a, b, k)) for a, b in zip(A, B)]


def secondary(args, line, rank, world, dev, peaks, peak_kind, model, w):
    """c0 line, Pearson GEMV (c1), KSG field (c2, full + like-for-like), bulk pairs (c4,
    full list), multi-reference cube (c3), reference default model (F3), CPU baselines."""
    import torch
    import paper_2307_02203_b200 as ndf
    from paper_2307_02203_b200 import _native as N
    from paper_2307_02203_b200 import workloads as W
    from concurrent.futures import ProcessPoolExecutor
    stream = torch.cuda.current_stream(dev)
    V = w.n_vertices
    shard = math.ceil(V / world)
    v0, v1 = min(V, rank * shard), min(V, (rank + 1) * shard)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    procs = os.cpu_count() or 1
    cpu = rank == 0 and world == 1 and not args.no_cpu
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    hbm = peaks.get("hbm_gbs", 6650.0)
    peak = peaks.get("bf16_tflops", 1590.0)

    def ev_ms(fn, reps, warm=1, flushing=True):
        out = []
        for i in range(warm + reps):
            if flushing:
                flush.fill_(float(i))
            t0.record(stream)
            fn()
            t1.record(stream)
            torch.cuda.synchronize()
            if i >= warm:
                out.append(t0.elapsed_time(t1))
        return statistics.mean(out)

    # ---- config 0: the CPU-runnable parity config (fp32), GPU vs CPU ----------------
    if rank == 0:
        from oracle import ndf_oracle as O
        w0 = W.CONFIGS[0]
        m0 = W.build_model(w0, seed=0, grid_init=1e-4).with_precision("fp32")
        f0 = W.generate_host(w0)
        ref0 = w0.ref_position()
        q_ms = ev_ms(lambda: ndf.reconstruct_field_device(m0, ref0, ndf.ROLE_MU, w0.dims), 10)
        gt_ms = ev_ms(lambda: ndf.ground_truth_field_device(
            f0, ndf.CorrelationMeasure("pearson"), "v", "v", ref0, w0.dims), 10)
        c0 = {"query_ms": q_ms, "gt_pearson_ms": gt_ms, "vertices": w0.n_vertices,
              "members": w0.members, "precision": "fp32 (exact path)"}
        if cpu:
            om0 = O.OracleModel(6, m0.grid_mu, m0.grid_nu, m0.weights, m0.biases, m0.spec.merge,
                                m0.spec.activation, m0.spec.head_kind)
            tc = time.perf_counter()
            O.reconstruct_field(om0, ref0, w0.dims)
            cq = (time.perf_counter() - tc) * 1e3
            tc = time.perf_counter()
            O.ground_truth_field(f0.member_grids("v"), "pearson", ref0, w0.dims)
            cg = (time.perf_counter() - tc) * 1e3
            c0["cpu_baseline"] = {"query_ms": cq, "gt_pearson_ms": cg, "cores": 1, "kind": "port",
                                  "sample": "full config-0 grid, oracle reconstruct_field and "
                                            "ground_truth_field(pearson), one process"}
        line["c0_cpu_config"] = c0
    # ---- ground-truth Pearson (c1): the fused one-pass field kernel, the public call
    # on a fresh ensemble, and the GEMV over a standardised copy Z ------------------
    ens = W.generate_device(w, dev)
    M = ens.member_count
    ref_vec = ens.X.reshape(M, -1)[:, w.ref_flat()].double().contiguous()
    outf = torch.empty(v1 - v0, dtype=torch.float32, device=dev)
    fms = max_over_ranks(ev_ms(lambda: N.call(
        "ndf_pearson_field", N.ptr(ens.X), M, V, 0, N.ptr(ref_vec), v0, v1, N.ptr(outf),
        N.stream_handle(dev)), args.steps, args.warmup), world)
    fbytes = 4.0 * M * (v1 - v0) + 4.0 * (v1 - v0)
    del outf
    torch.cuda.synchronize()
    Z, norm = ens.zscore()          # built once (allocation outside the timing below)
    zscore_ms = max_over_ranks(ev_ms(lambda: N.call(
        "ndf_zscore", N.ptr(ens.X), M, V, 0, V, N.ptr(Z), N.ptr(norm), N.stream_handle(dev)),
        3, 1), world)
    ref_flat = w.ref_flat()
    zref = Z[:, ref_flat].contiguous()
    out = torch.empty(v1 - v0, dtype=torch.float32, device=dev)
    gms = max_over_ranks(ev_ms(lambda: N.call(
        "ndf_pearson_gemv", N.ptr(Z), N.ptr(norm), M, V, N.ptr(zref), 0, v0, v1, N.ptr(out),
        N.stream_handle(dev)), args.steps, args.warmup), world)
    gbytes = 4.0 * M * (v1 - v0) + 4.0 * (v1 - v0) * 2
    gemv_gbs = gbytes / (gms * 1e-3) / 1e9
    zbytes = 8.0 * M * (v1 - v0) + 4.0 * (v1 - v0)
    del Z, norm, zref
    ens.drop_derived()

    def fresh():
        ens.drop_derived()
        ndf.ground_truth_field_device(ens, ndf.CorrelationMeasure("pearson"), "v", "v",
                                      w.ref_position(), w.dims, v0, v1)
    fresh_ms = max_over_ranks(ev_ms(fresh, 3), world)
    if rank == 0:
        fgbs = fbytes / (fms * 1e-3) / 1e9
        line["pearson_field"] = {
            "ms": fms, "bytes": fbytes, "achieved_gbs": fgbs, "peak_gbs": hbm,
            "frac": fgbs / hbm, "peak_kind": f"{peak_kind} hbm copy",
            "kernel": "ndf::pearson_field_kernel (+ pearson_ref_kernel)",
            "traffic": load_traffic().get("pearson_field_kernel"),
            "note": "one streaming read of X (fp64 shifted moments per column); what "
                    "ground_truth_field(pearson) runs on node-aligned grids",
            "fresh_public_call_ms": fresh_ms, "members": M, "vertices": v1 - v0,
            "roofline": {"bound": "hbm", "achieved": fgbs, "peak": hbm, "unit": "GB/s",
                         "frac": fgbs / hbm, "traffic": load_traffic().get("pearson_field_kernel"),
                         "bytes_basis": "4 M B read + 4 B written per vertex column"}}
        line["pearson_gemv"] = {
            "ms": gms, "bytes": gbytes, "achieved_gbs": gemv_gbs, "peak_gbs": hbm,
            "frac": gemv_gbs / hbm, "peak_kind": f"{peak_kind} hbm copy",
            "traffic": load_traffic().get("gemv_kernel"),
            "zscore_prep_ms": zscore_ms, "zscore_bytes": zbytes,
            "zscore_frac": zbytes / (zscore_ms * 1e-3) / 1e9 / hbm,
            "fresh_ensemble_ms": fresh_ms,
            "fresh_note": "public ground_truth_field_device on an ensemble with no cached Z",
            "members": M, "vertices": v1 - v0,
            "roofline": {"bound": "hbm", "achieved": gemv_gbs, "peak": hbm, "unit": "GB/s",
                         "frac": gemv_gbs / hbm, "traffic": load_traffic().get("gemv_kernel"),
                         "bytes_basis": "4 M B of Z read + 8 B per vertex (norm, out)"}}
    ens.drop_derived()
    del ens
    torch.cuda.empty_cache()
    # ---- KSG field on config 2: full field, and the CPU's own sample on both sides ----
    w2 = W.CONFIGS[2]
    ens2 = W.generate_device(w2, dev)
    M2 = ens2.member_count
    ref_vec = ens2.X.reshape(M2, -1)[:, w2.ref_flat()].double().contiguous()
    from paper_2307_02203_b200.measures import _KsgTables
    jit, psi = _KsgTables.get(dev, M2)
    mi = torch.empty(v1 - v0, dtype=torch.float32, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    psi_km = _KsgTables.psi_km(w2.ksg_k, M2)
    kfull = max_over_ranks(ev_ms(lambda: N.call(
        "ndf_ksg_ref_nodes", N.ptr(ens2.X), M2, V, N.ptr(ref_vec), v0, v1, w2.ksg_k, N.ptr(jit),
        N.ptr(psi), psi_km, None, N.ptr(mi), None, N.ptr(status), N.stream_handle(dev)),
        max(1, args.steps // 10), 1, flushing=False), world)
    pairs_s = V / (kfull * 1e-3)
    ksg = {"pairs_per_s": pairs_s, "unit": "pairs/s", "k": w2.ksg_k, "members": M2,
           "full_field_ms": kfull, "pairs": V,
           "note": "one launch over all 1.76 M config-2 vertices (measured, not extrapolated)"}
    if cpu:
        idx = np.random.default_rng(3).choice(V, size=args.cpu_ksg_pairs, replace=False)
        X2 = ens2.X.reshape(M2, -1)
        cols = X2[:, torch.from_numpy(idx).to(dev)].double().t().contiguous()   # (n, M) fp64
        mi_s = torch.empty(len(idx), dtype=torch.float32, device=dev)
        ks = ev_ms(lambda: N.call(
            "ndf_ksg_rows", N.ptr(ref_vec), 0, N.ptr(cols), M2, len(idx), w2.ksg_k, N.ptr(jit),
            N.ptr(psi), psi_km, None, N.ptr(mi_s), None, N.ptr(status), N.stream_handle(dev)),
            3, 1, flushing=False)
        Xh = cols.cpu().numpy()
        rate, kdt = cpu_ksg_rate(np.ascontiguousarray(np.column_stack([Xh.T, ref_vec.cpu().numpy()])),
                                 len(idx), np.arange(len(idx)), w2.ksg_k, procs)
        ksg["same_sample"] = {
            "vertices": len(idx), "gpu_pairs_per_s": len(idx) / (ks * 1e-3),
            "cpu_pairs_per_s": rate, "speedup_vs_cpu": len(idx) / (ks * 1e-3) / rate,
            "sample": f"{len(idx)} seeded-random config-2 vertices (rng 3) on both sides: GPU "
                      f"ndf_ksg_rows on the gathered columns, CPU oracle ksg_mi (scipy cKDTree, "
                      f"the reference algorithm) in {procs} processes ({kdt:.1f} s wall)"}
        ksg["cpu_pairs_per_s"] = rate
        ksg["speedup_vs_cpu"] = pairs_s / rate
        ksg["cpu_baseline"] = {"value": rate, "unit": "pairs/s", "cores": procs, "kind": "port",
                               "sample": ksg["same_sample"]["sample"]}
    tr = load_traffic()
    ksg["roofline"] = {"bound": "sm", "achieved": tr.get("ksg_kernel_sm_pct"), "peak": 100.0,
                       "unit": "% SM throughput (ncu)",
                       "frac": (tr.get("ksg_kernel_sm_pct") or 0.0) / 100.0 or None,
                       "traffic": tr.get("ksg_kernel_16384_pairs"),
                       "source": "profiles/r02/prof_ksg.txt (ncu --set full, 16,384 c2 pairs)",
                       "note": "fp64 compare / select work (exact k-NN scans, bitonic sorts, binary "
                               "searches): no FLOP or byte roofline applies; SM throughput is the "
                               "north_star's KSG evidence"}
    if rank == 0:
        line["ksg_mi"] = ksg
    # ---- config 4: bulk estimator pairs (Pearson + KSG), the full 2^22 list ----------
    n_pairs = args.c4_pairs
    pa_all, pb_all = W.pair_list(W.CONFIGS[4], count=n_pairs, seed=2)
    ps = math.ceil(n_pairs / world)
    p0, p1 = min(n_pairs, rank * ps), min(n_pairs, (rank + 1) * ps)
    ens2.vertex_major()
    ndf.pair_estimators_device(ens2, "v", pa_all[p0:p0 + 1024], pb_all[p0:p0 + 1024],
                               k=W.CONFIGS[4].ksg_k)
    torch.cuda.synchronize()
    res = {}

    def c4():
        res["r"] = ndf.pair_estimators_device(ens2, "v", pa_all[p0:p1], pb_all[p0:p1],
                                              k=W.CONFIGS[4].ksg_k)
        if world > 1:                      # result assembly inside the timed region
            from paper_2307_02203_b200.parallel import gather_shards
            res["g"] = {k: gather_shards(v, n_pairs) for k, v in res["r"].items()}
    c4_ms = max_over_ranks(ev_ms(c4, 1, 0, flushing=False), world)
    res.clear()
    c4l = {"pairs": n_pairs, "ms": c4_ms, "pairs_per_s": n_pairs / (c4_ms * 1e-3),
           "estimators": ["pearson", "ksg_mi"], "k": W.CONFIGS[4].ksg_k,
           "note": "the seeded config-4 pair list (half uniform, half within +-16 cells), "
                   "public pair_estimators_device; vertex-major copy built before timing"}
    if cpu:
        nc = min(args.cpu_c4_pairs, n_pairs)
        sel = np.random.default_rng(4).choice(n_pairs, nc, replace=False)
        X2 = ens2.X.reshape(M2, -1)
        A = X2[:, torch.from_numpy(pa_all[sel]).to(dev)].double().t().cpu().numpy()
        B = X2[:, torch.from_numpy(pb_all[sel]).to(dev)].double().t().cpu().numpy()
        parts = [(A[i::procs * 2], B[i::procs * 2], W.CONFIGS[4].ksg_k) for i in range(procs * 2)]
        tc = time.perf_counter()
        with ProcessPoolExecutor(max_workers=procs) as ex:
            list(ex.map(_c4_cpu_chunk, parts))
        cdt = time.perf_counter() - tc
        c4l["cpu_pairs_per_s"] = nc / cdt
        c4l["speedup_vs_cpu"] = c4l["pairs_per_s"] / c4l["cpu_pairs_per_s"]
        c4l["cpu_sample"] = (f"{nc} seeded pairs of the list, oracle pearson_rowwise + ksg_mi "
                             f"(scipy cKDTree) in {procs} processes, {cdt:.1f} s wall")
        c4l["cpu_baseline"] = {"value": nc / cdt, "unit": "pairs/s", "cores": procs, "kind": "port",
                               "sample": c4l["cpu_sample"]}
    tr = load_traffic()
    c4l["roofline"] = {"bound": "sm", "achieved": tr.get("ksg_kernel_pairs_sm_pct"), "peak": 100.0,
                       "unit": "% SM throughput (ncu)",
                       "frac": (tr.get("ksg_kernel_pairs_sm_pct") or 0.0) / 100.0 or None,
                       "kernel": "ndf::ksg_kernel<9> (pairs mode), ~99% of the step",
                       "source": "profiles/r02/prof_pairs_ksg.txt (ncu --set full)",
                       "pearson_pairs": {"bound": "hbm", "unit": "% of DRAM peak (ncu)",
                                         "achieved": tr.get("pearson_pairs_dram_pct"),
                                         "source": "profiles/r02/prof_pairs_pearson.txt"}}
    if rank == 0:
        line["c4_bulk_pairs"] = c4l
    ens2.drop_derived()
    # ---- F2's caller: training targets (training.py:111-119) of uniform off-grid pairs --
    if rank == 0:
        tp = 1 << 16
        trng = np.random.default_rng(12)
        tmu, tnu = trng.uniform(-1.0, 1.0, (tp, 3)), trng.uniform(-1.0, 1.0, (tp, 3))
        tm = ndf.CorrelationMeasure("ksg_mi", ksg_k=W.CONFIGS[4].ksg_k)
        tpe = ndf.CorrelationMeasure("pearson")
        ndf.targets_device(ens2, tpe, "v", "v", tmu, tnu)   # warm-up: builds the vertex-major copy
        t_ms = ev_ms(lambda: ndf.targets_device(ens2, tm, "v", "v", tmu, tnu), 1, 0, flushing=False)
        tp_ms = ev_ms(lambda: ndf.targets_device(ens2, tpe, "v", "v", tmu, tnu), 3, 1, flushing=False)
        tl = {"pairs": tp, "ksg_ms": t_ms, "pearson_ms": tp_ms, "pairs_per_s": tp / (t_ms * 1e-3),
              "k": W.CONFIGS[4].ksg_k,
              "note": "public targets_device over uniform off-grid position pairs of the config-2 "
                      "ensemble: fp64 trilinear samples from the variable's vertex-major copy (built "
                      "once per variable, in the warm-up) into HBM, one KSG (or Pearson) launch"}
        if cpu:
            nc = min(args.cpu_c4_pairs, tp)
            # the samples the reference's sample_many would produce (bit-identical, tests)
            A = ens2.sample_many(tmu[:nc]).cpu().numpy()
            B = ens2.sample_many(tnu[:nc]).cpu().numpy()
            parts = [(A[i::procs * 2], B[i::procs * 2], W.CONFIGS[4].ksg_k) for i in range(procs * 2)]
            tc = time.perf_counter()
            with ProcessPoolExecutor(max_workers=procs) as ex:
                list(ex.map(_c4_cpu_chunk, parts))
            cdt = time.perf_counter() - tc
            tl["cpu_baseline"] = {"value": nc / cdt, "unit": "pairs/s", "cores": procs, "kind": "port",
                                  "sample": f"{nc} of the pairs: oracle pearson_rowwise + ksg_mi per "
                                            f"pair (scipy cKDTree) in {procs} processes on their "
                                            f"samples ({cdt:.1f} s wall; sampling untimed)"}
            tl["speedup_vs_cpu"] = tl["pairs_per_s"] / tl["cpu_baseline"]["value"]
        line["training_targets"] = tl
    del ens2
    torch.cuda.empty_cache()
    # ---- config 3: 64-reference cube, both heads, the benched precision ---------------
    w3 = W.CONFIGS[3]
    refs = W.reference_vertices(w3, count=64, seed=1)
    pos = np.stack([np.array([2.0 * i / (n - 1) - 1.0 for i, n in
                              zip((v % w3.dims[0], (v // w3.dims[0]) % w3.dims[1],
                                   v // (w3.dims[0] * w3.dims[1])), w3.dims)]) for v in refs])
    prec3 = model.spec.precision if model.spec.precision != "fp32" else "bf16"
    models = [W.build_model(w3, seed=0, grid_init=1e-4).with_precision(prec3),
              ndf.NdfModel.build(
                  ndf.ModelSpec.baseline(w3.dims, w3.latent_factor, measure_kind="ksg_mi",
                                         precision=prec3), seed=1)]
    cube = torch.empty((64, v1 - v0), dtype=torch.float16, device=dev)

    def c3():
        for m3 in models:
            ndf.reconstruct_multi_device(m3, pos, ndf.ROLE_MU, w3.dims, v0, v1, out=cube)
            if world > 1:                  # the 64 x 1.76 M cube assembled on every rank
                from paper_2307_02203_b200.parallel import gather_columns
                gather_columns(cube, V)
    c3_ms = max_over_ranks(ev_ms(c3, max(1, args.steps // 5), 1, flushing=False), world)
    if rank == 0:
        pairs3 = 2 * 64 * V
        tf3 = FLOP_PER_PAIR * pairs3 / (c3_ms * 1e-3) / 1e12
        sm_count = torch.cuda.get_device_properties(dev).multi_processor_count
        sm_hz = ((line.get("clocks") or {}).get("sm_mhz") or 1965.0) * 1e6
        sfu3 = SFU_OPS_PER_PAIR * pairs3 / (SFU_PER_CLK_SM * sm_count * sm_hz) * 1e3
        line["c3_multi_ref"] = {"refs": 64, "heads": 2, "pairs": pairs3, "ms": c3_ms,
                                "precision": prec3,
                                "pairs_per_s": pairs3 / (c3_ms * 1e-3),
                                "roofline": {"bound": "tensor", "achieved": tf3, "peak": peak,
                                             "unit": "TFLOP/s", "frac": tf3 / peak,
                                             "flop_basis": "algorithmic 93,952 FLOP per pair",
                                             "sfu_floor_ms": sfu3, "sfu_frac": sfu3 / c3_ms},
                                "output": "fp16 cube 64 x 1.76M per head"}
    del cube, models
    # ---- SURVEY row A2 standalone: the positional encoder (K1) over the config-1 grid
    # (NdfModel.embed_nodes -> ndf_embed_nodes); the query kernels fuse it ------------------
    emb_ms = max_over_ranks(ev_ms(lambda: model.embed_nodes("mu", w.dims, v0, v1),
                                  max(1, args.steps // 2)), world)
    if rank == 0:
        eb = 4.0 * 55 * (v1 - v0)
        egbs = eb / (emb_ms * 1e-3) / 1e9
        line["encoder_k1"] = {
            "ms": emb_ms, "vertices": v1 - v0, "features": 55,
            "roofline": {"bound": "hbm", "achieved": egbs, "peak": hbm, "unit": "GB/s",
                         "frac": egbs / hbm, "traffic": load_traffic().get("embed_nodes_kernel"),
                         "bytes_basis": "220 B of fp32 features written per node (the latent "
                                        "grid, 1.8 MB, and the axis tables stay in L2)"},
            "kernel": "ndf::embed_nodes_kernel (+ embed_axis_kernel)",
            "note": "bit-identical to the reference's fp64 embed; L1-bound on the latent "
                    "corner reads (profiles/r02/prof_embed.txt)"}
    torch.cuda.empty_cache()
    # ---- the reference's own default architecture (HashGrid + encoder
    # MLPs, exact fp32 path) queried over the config-1 grid ------------------------------
    mref = ndf.NdfModel.build(ndf.ModelSpec.reference_default(), seed=0)
    outr = torch.empty(v1 - v0, dtype=torch.float32, device=dev)
    f3_ms = max_over_ranks(ev_ms(lambda: ndf.reconstruct_field_device(
        mref, w.ref_position(), ndf.ROLE_MU, w.dims, v0, v1, out=outr),
        max(1, args.steps // 5)), world)
    if rank == 0:
        spec = mref.spec
        line["f3_reference_default"] = {
            "ms": f3_ms, "vertices": V, "precision": "fp32 (exact, matmul_exact order)",
            "model": f"reference ModelSpec(): {spec.levels}-level HashGrid 2^{spec.log2_table_size}"
                     f"x{spec.features_per_level}, encoders {spec.encoder_widths()}, decoder "
                     f"{spec.decoder_widths()}, {spec.merge} merge, snake_alt, linear head"}
    del outr, mref
    # ---- the /api/reconstruct binary data plane (body + value-range
    # headers in pinned host memory), host wall clock per call like e2e --------------------
    if rank == 0:
        for _ in range(args.warmup):
            ndf.reconstruct_response(model, w.ref_position(), ndf.ROLE_MU, w.dims)
        ts = []
        for _ in range(args.steps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            resp = ndf.reconstruct_response(model, w.ref_position(), ndf.ROLE_MU, w.dims)
            ts.append((time.perf_counter() - t0) * 1e3)
            del resp
        line["f4_response"] = {
            "ms": statistics.mean(ts), "bytes": 4 * V,
            "note": "reconstruct_response (service.py:392-410 without HTTP): one query launch "
                    "(ndf_query_grid_stats) stores the fp32 body into pinned host memory and "
                    "reduces the X-Value-Min / X-Value-Max range in its epilogue"}
    # ---- CPU baseline of the headline (rank 0, N=1 only): the full config-1 grid -------
    if cpu:
        m32 = model.with_precision("fp32")
        with oracle_pool(m32, w, procs) as pool:
            sample = cpu_sample_size(m32, w, procs, pool, args.cpu_sample, args.ref_step_s)
            per_v, dt = cpu_query_rate(m32, w, sample, procs, pool=pool)
        cpu_ms = per_v * V * 1e3
        scope = "the full grid" if sample == V else f"{sample} seeded vertices, extrapolated"
        line["cpu_baseline"] = {
            "value": cpu_ms, "unit": "ms", "cores": procs, "kind": "port",
            "sample": f"config 1 via oracle/ndf_oracle.py reconstruct_field (reference einsum "
                      f"order) over {scope} in {procs} processes, {dt:.2f} s wall"}
        if "c3_multi_ref" in line:
            c3l = line["c3_multi_ref"]
            c3l["cpu_baseline"] = {"ms": per_v * c3l["pairs"] * 1e3, "cores": procs, "kind": "port",
                                   "sample": "config-1 per-vertex CPU rate above x 128 "
                                             "reference-head queries (SURVEY 8(d) c3)"}
            c3l["speedup_vs_cpu"] = c3l["cpu_baseline"]["ms"] / c3l["ms"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--precision", choices=["bf16", "fp16", "fp32"], default="bf16")
    ap.add_argument("--quick", action="store_true", help="query only (profiling runs)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=1760000)
    ap.add_argument("--cpu-ksg-pairs", type=int, default=4096)
    ap.add_argument("--cpu-c4-pairs", type=int, default=4096)
    ap.add_argument("--ref-sample", type=int, default=1760000)
    ap.add_argument("--ref-step-s", type=float, default=4.0,
                    help="cap on one CPU step; larger grids are sampled and extrapolated")
    ap.add_argument("--c4-pairs", type=int, default=1 << 22)
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
