"""Benchmark: ROIs/s of full 3-D shape coefficients on KiTS19-shaped masks.

Contract (driver): `python bench.py --gpus N --steps K --warmup W` prints ONE
JSON line on rank 0.  N>1 runs under torchrun, one rank per GPU; every rank
processes its own ROIs (ROI-batch sharding: independent masks, no data-path
collective -> "scaling": "weak"); the timed region is bracketed by a barrier
and torch.cuda.synchronize() and the reported time is the max over ranks.

Workload (default, BASELINE.json configs[3]): C4, the batch of 300 varied
KiTS19-shaped masks (512x512x[200..700], seed 2025); each rank
takes its LPT share.  One step = one call of the batch entry on B (--batch,
default 64) ROIs of the rank's share, cycling through it, so consecutive
steps see different masks.  Every mask is staged in HBM before timing; every
mask is larger than the 126 MB L2 or, cycling 300 distinct masks, evicted
long before it comes back, so no L2 flush is needed.  C2 (configs[1], one
512x512x600 mask at 0.8x0.8x1.0 mm) is measured the same way beside it
(key "c2").  --workload c1|c2|c3|c5 selects another SURVEY.md 8(d) config.

  value      device-resident throughput: K batch calls of B ROIs
             (sc_calculate_coefficients_device_batch, 32 pipeline slots),
             CUDA events on the caller's stream (each call is ordered against
             it and synchronous).
  e2e        the same metric through the C ABI with HOST (pinned) masks:
             sc_calculate_coefficients_batch, B ROIs per step; the host scans
             every mask byte for the occupied slab and only the slab crosses
             PCIe; every result record is read back.
  roi_ceiling  per-ROI HBM bound: mask bytes / measured copy bandwidth vs the
             measured time per ROI.
  roofline   the dominant kernel of the batch path, the HBM-bound TMA pack
             (pack_bits_tma: mask bytes read once per launch), timed with CUDA
             events around the kernel; roofline_pass1 = the FP32 diameter
             pass (8 flop per evaluated pair vs the FP32 rate measured by
             sc_probe_fp32_peak on this GPU).
  dominant_kernel  the largest single kernel of this workload's one-ROI call
             (C3: mc_cells), its share, its bound and its committed ncu counters.
  cpu_baseline  the reference itself (shapecore, numba, installed under
             baseline/_ref) on all host cores on a bounded sample of the
             workload; the C port in oracle/ when the install is missing.

`--impl reference` times the reference's CPU path alone (rank 0; other ranks
exit 0): extract_features(vol, resolve_backend("parallel")) per ROI
(features.py:224-265, dispatch.py:103-146), plus the "sequential" backend on
C1 (PyRadiomics' shape class is single-threaded).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ROIs/sec full 3D shape coefficients (KiTS19-shaped masks) at 1/2/4/8 B200"
UNIT = "ROIs/s"

# SURVEY.md 8(d) configurations.  The default (headline) is c4, the batch of
# varied KiTS19-shaped masks; the others are selectable with --workload.
WORKLOADS = {
    "c1": "C1 synthetic 64^3 sphere mask (r=24, spacing 1 mm, V=10824; the reference's own "
          "CPU-runnable case)",
    "c2": "C2 KiTS19-shaped synthetic kidney+tumor mask 512x512x600 uint8 at 0.8x0.8x1.0 mm "
          "(tumor 30 mm, V=73406)",
    "c3": "C3 noisy-boundary ellipsoid 512^3 at 1 mm (sigma 0.02, seed 1234, V=1963474, "
          "1.93e12 pairs)",
    "c4": "C4 batch of 300 varied KiTS19-shaped masks (512x512x[200..700] uint8, in-plane "
          "spacing 0.6-0.9 mm, tumour 10-75 mm, seed 2025), LPT-sharded across GPUs",
    "c5": "C5 thin slab 512x512x24 at 0.5x0.5x5 mm, 400 blobs (seed 7, V=127664)",
}


def workload_params(name, rank=0, world=1):
    """[(generator, spacing)] of this rank's ROIs (masks are generated lazily,
    one at a time, so 300 C4 masks never sit in host memory together)."""
    from paper_2510_02894_b200 import sharding, synth

    if name == "c1":
        return [(lambda: synth.synth_mask("sphere", (64, 64, 64), radius=24), (1.0, 1.0, 1.0))]
    if name == "c2":
        return [(lambda: synth.kits_like(512, 512, 600, (0.8, 0.8, 1.0), 30.0), (0.8, 0.8, 1.0))]
    if name == "c3":
        return [(lambda: synth.noisy_ellipsoid(512, 0.02, 1234), (1.0, 1.0, 1.0))]
    if name == "c5":
        return [(lambda: synth.thin_slab(), (0.5, 0.5, 5.0))]
    if name == "c4":
        params = synth.kits_batch_params(300, 2025)
        # cost: streamed voxels + (surface ~ tumour/kidney size)^2 pairs
        costs = [sharding.roi_cost(int((p["tumor_mm"] / p["sp"][0]) ** 3 * 4.2 + 2.6e5),
                                   p["nx"] * p["ny"] * p["nz"]) for p in params]
        mine = sharding.assign_rois(costs, world)[rank]
        return [((lambda p=params[i]: synth.kits_from_params(p)), tuple(params[i]["sp"]))
                for i in mine]
    raise SystemExit(f"unknown workload {name}")


def load_workload(name, rank=0, world=1):
    """[(mask (nz,ny,nx) uint8, spacing)] for this rank, plus a config dict
    (host masks; tools/ use this)."""
    rois = [(g(), sp) for g, sp in workload_params(name, rank, world)]
    cfg = {
        "workload": WORKLOADS[name],
        "name": name,
        "roi_bytes_mean": sum(m.size for m, _ in rois) / max(1, len(rois)),
        "rois_per_rank": len(rois),
    }
    return rois, cfg


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0}, "fallback (B200_PROFILING.md)"


def ncu_traffic():
    """Per-launch DRAM bytes of the dominant kernels from the committed ncu
    summary (profiles/ncu_summary.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as fh:
            return json.load(fh).get("dram_bytes_per_launch", {})
    except (OSError, ValueError):
        return {}


class ClockSampler:
    """SM clock and throttle reasons sampled through NVML every ~2 ms while the
    timed region runs (the region is tens of ms, too short for nvidia-smi -lms)."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, cuda_index: int):
        self.idx = cuda_index
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self.thread = None
        self.h = None

    def _handle(self):
        import pynvml
        import torch

        pynvml.nvmlInit()
        p = torch.cuda.get_device_properties(self.idx)
        try:
            bus = f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
            return pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            return pynvml.nvmlDeviceGetHandleByIndex(self.idx)

    def _run(self):
        import pynvml

        while not self._stop.is_set():
            try:
                self.samples.append(pynvml.nvmlDeviceGetClockInfo(self.h, pynvml.NVML_CLOCK_SM))
                r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        try:
            import pynvml

            self.h = self._handle()
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.thread = threading.Thread(target=self._run, daemon=True)
            self.thread.start()
        except Exception as exc:  # NVML missing: report, do not fail the bench
            self.reasons.add(f"unsampled: {exc}")
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self.thread:
            self.thread.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz,
                    "reasons": sorted(self.reasons) or ["unsampled"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def dist_setup(n_gpus):
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(world, value):
    if world == 1:
        return value
    import torch
    import torch.distributed as dist

    t = torch.tensor([value], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def reference_module():
    """The reference itself (shapecore: Python + numba), installed under
    baseline/_ref by build(); None when the install is missing."""
    path = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(path, "shapecore")):
        return None
    if path not in sys.path:
        sys.path.insert(0, path)
    try:
        import shapecore

        return shapecore
    except Exception:  # numba missing or broken: fall back to the C port
        return None


def reference_roi_seconds(ref, mask, sp, backend="parallel"):
    """One ROI through the reference's public path: MaskVolume ->
    extract_features(vol, resolve_backend(backend, workers=all host cores))
    (features.py:224-265, dispatch.py:103-146).  Returns (seconds, record)."""
    nz, ny, nx = mask.shape
    vol = ref.MaskVolume(dims=(nx, ny, nz), spacing=tuple(float(v) for v in sp),
                         data=mask.reshape(-1))
    sel = ref.resolve_backend(backend, workers=os.cpu_count()) if backend == "parallel" \
        else ref.resolve_backend(backend)
    t0 = time.perf_counter()
    feats, _ = ref.extract_features(vol, sel)
    return time.perf_counter() - t0, feats.to_dict()


def reference_warmup(ref, n=1):
    """JIT-compile (numba, cache=True) and warm the reference on the C1 sphere."""
    from paper_2510_02894_b200 import synth

    c1 = synth.synth_mask("sphere", (64, 64, 64), radius=24)
    for _ in range(max(1, n)):
        reference_roi_seconds(ref, c1, (1.0, 1.0, 1.0), "parallel")
        reference_roi_seconds(ref, c1, (1.0, 1.0, 1.0), "sequential")


def reference_layer():
    import numba

    try:
        return numba.threading_layer()
    except Exception:
        return "unknown"


def port_roi_seconds(mask, sp):
    """The C restatement of the reference (oracle/, OpenMP strip-parallel
    diameters, serial MC) on one ROI: the fallback CPU baseline."""
    from oracle import oracle

    t0 = time.perf_counter()
    oracle.extract_features(mask, sp, threads=0, with_active=False)
    return time.perf_counter() - t0, oracle.max_threads()


def cpu_baseline_sample(gens, max_seconds, max_rois):
    """Bounded sample of the workload on the host cores: the reference when
    installed, else the C port.  Returns the cpu_baseline object."""
    ref = reference_module()
    times = []
    t_start = time.perf_counter()
    if ref is not None:
        import numba

        reference_warmup(ref)
        for i in range(max_rois):
            g, sp = gens[i % len(gens)]
            dt, _ = reference_roi_seconds(ref, g(), sp)
            times.append(dt)
            if time.perf_counter() - t_start > max_seconds:
                break
        per = statistics.mean(times)
        return {"value": 1.0 / per, "unit": UNIT, "cores": int(numba.get_num_threads()),
                "kind": "reference",
                "sample": f"{len(times)} ROI(s) of the workload through the reference itself "
                          "(baseline/_ref shapecore: extract_features(vol, resolve_backend("
                          "'parallel', workers=os.cpu_count())), numba threading layer "
                          f"{reference_layer()}), after a JIT warm-up",
                "seconds_per_roi": per}
    threads = 1
    for i in range(max_rois):
        g, sp = gens[i % len(gens)]
        dt, threads = port_roi_seconds(g(), sp)
        times.append(dt)
        if time.perf_counter() - t_start > max_seconds:
            break
    per = statistics.mean(times)
    return {"value": 1.0 / per, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{len(times)} ROI(s) through oracle/shape_oracle.c (reference algorithm "
                      "restated in C: serial canonical MC, strip-parallel fp64 diameters); "
                      "baseline/_ref missing", "seconds_per_roi": per}


def run_reference(args):
    """The reference's own CPU path (shapecore, numba) on the host cores.
    Rank 0 alone runs and prints; other ranks exit 0 without work."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return 0
    gens = workload_params(args.workload, 0, 1)
    ref = reference_module()
    extra = {}
    if ref is None:
        kind, cores = "port", 1
        times = []
        t0 = time.perf_counter()
        for i in range(args.steps):
            g, sp = gens[i % len(gens)]
            dt, cores = port_roi_seconds(g(), sp)
            times.append(dt)
            if time.perf_counter() - t0 > args.cpu_seconds:
                break
        sample = "oracle/shape_oracle.c, the C restatement (baseline/_ref missing)"
    else:
        import numba

        kind, cores = "reference", int(numba.get_num_threads())
        # W warm-up steps: JIT compile + numba cache on the C1 sphere (a full
        # C4 ROI costs seconds on the CPU; the warm-up only has to compile).
        reference_warmup(ref, args.warmup)
        times = []
        t0 = time.perf_counter()
        for i in range(args.steps):
            g, sp = gens[i % len(gens)]
            dt, _ = reference_roi_seconds(ref, g(), sp)
            times.append(dt)
            if time.perf_counter() - t0 > args.cpu_seconds:
                break
        # PyRadiomics' shape class is single-threaded: the
        # reference's "sequential" backend on C1, for the record.
        from paper_2510_02894_b200 import synth

        c1 = synth.synth_mask("sphere", (64, 64, 64), radius=24)
        seq = [reference_roi_seconds(ref, c1, (1.0, 1.0, 1.0), "sequential")[0] for _ in range(5)]
        par = [reference_roi_seconds(ref, c1, (1.0, 1.0, 1.0), "parallel")[0] for _ in range(5)]
        extra = {"c1_sequential": {"value": 1.0 / statistics.median(seq), "unit": UNIT,
                                   "cores": 1, "note": "C1 64^3 sphere, backend 'sequential', "
                                                       "median of 5"},
                 "c1_parallel": {"value": 1.0 / statistics.median(par), "unit": UNIT,
                                 "cores": cores, "note": "C1, backend 'parallel', median of 5"},
                 "numba_threading_layer": reference_layer(), "host_cpu_count": os.cpu_count()}
        sample = ("the reference itself: baseline/_ref shapecore (pip install of "
                  "/root/reference/pkg), extract_features(vol, resolve_backend('parallel', "
                  f"workers=os.cpu_count())) per ROI, numba layer {reference_layer()}")
    per = statistics.mean(times)
    value = 1.0 / per
    cfg = {"workload": WORKLOADS[args.workload], "name": args.workload,
           "global_batch": 1, "parallelism": "host cores (numba prange)" if kind == "reference"
           else "host cores (OpenMP)",
           "sample_rois": len(times), "l2": "n/a (CPU)"}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference",
        "n_gpus": world, "steps": len(times), "warmup": args.warmup,
        "ms_per_step": per * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u8 mask / fp64 (reference arithmetic)",
        "data": "synthetic", "config": cfg,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
                         "sample": f"{len(times)} ROI(s) of the workload (one per step, "
                                   f"distinct masks) through {sample}; time-capped at "
                                   f"{args.cpu_seconds:.0f}s"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    line.update(extra)
    print(json.dumps(line), flush=True)
    return 0


def stage_on_device(gens, dev, keep_host):
    """Generate the rank's masks one at a time and copy each to HBM; keep the
    first `keep_host` on the host in pinned memory (the e2e leg)."""
    import torch

    d_masks, host = [], []
    for i, (g, sp) in enumerate(gens):
        m = g()
        t = torch.from_numpy(m)
        if i < keep_host:
            t = t.pin_memory()
            host.append(t.numpy())
        d_masks.append(t.to(f"cuda:{dev}", non_blocking=False))
    return d_masks, host


def timed_batches(sc, _native, d_masks, sps, B, K, W, stream, world):
    """W warm-up and K timed steps; step k = one device-batch call on ROIs
    [(k*B + i) % n].  Returns (ms max over ranks, launches, outputs of the
    timed steps, clocks)."""
    import torch

    n = len(d_masks)

    def step(k):
        idx = [(k * B + i) % n for i in range(B)]
        return idx, sc.calculate_coefficients_device_batch([d_masks[i] for i in idx],
                                                           [sps[i] for i in idx], stream=stream)

    for k in range(W):
        step(k)
    torch.cuda.synchronize()
    clocks = ClockSampler(torch.cuda.current_device())
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = _native.launch_count()
    barrier(world)
    torch.cuda.synchronize()
    clocks.__enter__()
    ev0.record(stream)
    outs = [step(W + k) for k in range(K)]
    ev1.record(stream)
    torch.cuda.synchronize()
    clocks.__exit__(None, None, None)
    barrier(world)
    launches = _native.launch_count() - launches0
    return max_over_ranks(world, ev0.elapsed_time(ev1)), launches, outs, clocks


def pack_batch_ms(sc, _native, d_masks, sps, B, stream):
    """Milliseconds per ROI of a B-ROI device batch that enqueues only the
    first two kernels per ROI (init_stats + the pack): the pack's launch
    duration as the batch runs it.  Best of 3 (after one warm-up batch)."""
    import torch

    n = len(d_masks)
    ms = [d_masks[i % n] for i in range(B)]
    ss = [sps[i % n] for i in range(B)]
    best = float("inf")
    with _native.thread_options(debug_stages=2):
        for r in range(4):
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            ev0.record(stream)
            try:
                sc.calculate_coefficients_device_batch(ms, ss, stream=stream)
            except Exception:  # a cut pipeline's records are meaningless
                pass
            ev1.record(stream)
            torch.cuda.synchronize()
            if r:
                best = min(best, ev0.elapsed_time(ev1) / B)
    return best


def check_repeats(outs):
    """Results of the same mask must be identical wherever it recurs."""
    seen = {}
    for idx, recs in outs:
        for i, r in zip(idx, recs):
            d = r.to_dict()
            assert seen.setdefault(i, d) == d, f"ROI {i}: results differ between steps"
    return seen


def kernel_times(sc, _native, d_mask, sp, stream, reps, dev, **opts):
    """Per-stage CUDA-event times (option stage_times=2) of single calls on
    one ROI: medians over `reps` calls, plus the diagnostics and record."""
    kt = {k: [] for k in _native.KERNEL_TIME_NAMES}
    with _native.thread_options(stage_times=2, **opts):
        sc.calculate_coefficients_device(d_mask, sp, stream=stream)  # captures its graph
        for _ in range(reps):
            c = sc.calculate_coefficients_device(d_mask, sp, stream=stream)
            for k, v in _native.last_kernel_times(dev).items():
                kt[k].append(v)
    med = {k: statistics.median(v) for k, v in kt.items() if v}
    return med, _native.last_diagnostics(dev), c


def run_ours(args):
    import torch

    import paper_2510_02894_b200 as sc
    from paper_2510_02894_b200 import _native

    world, rank, local = dist_setup(args.gpus)
    dev = torch.cuda.current_device()
    # The host slab scan of the e2e leg uses a share of the host cores per rank
    # (one process per GPU on one node).
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", str(world)))
    host_threads = max(1, (os.cpu_count() or 1) // max(1, local_world))
    _native.set_option("host_threads", min(32, host_threads))
    gens = workload_params(args.workload, rank, world)
    sps = [sp for _, sp in gens]
    n_host = min(len(gens), args.e2e_masks)
    d_masks, h_masks = stage_on_device(gens, dev, n_host)
    roi_bytes = [m.numel() for m in d_masks]
    stream = torch.cuda.Stream()
    B, K = args.batch, args.steps
    W = max(args.warmup, 3)
    peaks, peak_kind = measured_peaks()
    hbm = peaks["hbm_gbs"]

    # ---- device-resident throughput (value) ----
    dev_ms, launches, outs, clocks = timed_batches(sc, _native, d_masks, sps, B, K, W, stream,
                                                   world)
    value = world * B * K / (dev_ms / 1e3)
    recs = check_repeats(outs)
    us_roi = dev_ms * 1e3 / (B * K)
    step_bytes = sum(roi_bytes[(k * B + i) % len(d_masks)]
                     for k in range(W, W + K) for i in range(B)) / (B * K)
    ceiling_us = step_bytes / (hbm * 1e3)

    def ceiling(us, nbytes):
        return {"bytes_per_roi": nbytes, "hbm_gbs": hbm, "peak_kind": peak_kind,
                "ceiling_us_per_roi": nbytes / (hbm * 1e3), "measured_us_per_roi": us,
                "frac": nbytes / (hbm * 1e3) / us,
                "note": "every mask byte read once from HBM at the measured copy bandwidth: "
                        "the per-ROI floor of the whole pipeline"}

    # ---- C2 side by side (BASELINE.json configs[1]) ----
    side = None
    if args.workload == "c4" and not args.no_side:
        g2 = workload_params("c2")
        d2, _ = stage_on_device(g2, dev, 0)
        ms2, _, outs2, _ = timed_batches(sc, _native, d2, [g2[0][1]], B, K, W, stream, world)
        check_repeats(outs2)
        u2 = ms2 * 1e3 / (B * K)
        # the marching-cubes stage of one C2 call (pack + mc_cells, CUDA
        # events at every stage) against HBM: mask bytes / stage time
        med2, _, _ = kernel_times(sc, _native, d2[0], g2[0][1], stream,
                                  max(3, min(K, 10)), dev)
        mc_s = (med2["pack_ms"] + med2["mc_ms"]) / 1e3
        side = {"workload": WORKLOADS["c2"], "value": world * B * K / (ms2 / 1e3), "unit": UNIT,
                "us_per_roi": u2, "roi_ceiling": ceiling(u2, d2[0].numel()),
                "protocol": "same as value: K batch calls of B ROIs (the C2 mask repeated)",
                "mc_stage": {"pack_ms": med2["pack_ms"], "mc_ms": med2["mc_ms"],
                             "achieved_gbs": d2[0].numel() / mc_s / 1e9,
                             "frac_hbm": d2[0].numel() / mc_s / 1e9 / hbm,
                             "note": "single call: 128-bit-load pack + mc_cells, mask bytes / "
                                     "(pack + mc) time"}}
        del d2

    # ---- per-kernel times (single calls, CUDA events at every stage) ----
    i0 = max(range(len(d_masks)), key=lambda i: roi_bytes[i]) if args.workload != "c4" else 0
    d0, sp0 = d_masks[i0], sps[i0]
    reps = max(3, min(K, 20))
    med, diag, c = kernel_times(sc, _native, d0, sp0, stream, reps, dev)
    assert c.to_dict() == recs.get(i0, c.to_dict())
    # the batch path's pack (TMA bulk copy + fused bbox) timed the same way
    med_tma, _, c_tma = kernel_times(sc, _native, d0, sp0, stream, reps, dev,
                                     pack_tma_single=1, fused_bbox_single=1)
    assert c_tma.to_dict() == c.to_dict()
    # all pairs evaluated (no pruning): the brute-force pass-1 roofline
    bf_reps = 3 if args.workload == "c3" else max(3, reps // 2)
    bf_med, bf_diag, c_bf = kernel_times(sc, _native, d0, sp0, stream, bf_reps, dev, prune=0)
    assert c_bf.to_dict() == c.to_dict(), "pruned and all-pairs results differ"
    single_ms = []
    for _ in range(reps):
        t0 = time.perf_counter()
        sc.calculate_coefficients_device(d0, sp0, stream=stream)
        single_ms.append((time.perf_counter() - t0) * 1e3)

    # ---- end to end through the C ABI from pinned host memory (e2e) ----
    def e2e_run(opts):
        with _native.thread_options(**opts):
            hs = [h_masks[i % n_host] for i in range(B)]
            hsp = [sps[i % n_host] for i in range(B)]
            sc.calculate_coefficients_batch(hs, hsp, device=dev)  # warm-up
            barrier(world)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            e_outs = []
            for k in range(K):
                idx = [(k * B + i) % n_host for i in range(B)]
                e_outs.append((idx, sc.calculate_coefficients_batch(
                    [h_masks[i] for i in idx], [sps[i] for i in idx], device=dev)))
            torch.cuda.synchronize()
            s = max_over_ranks(world, time.perf_counter() - t0)
            barrier(world)
        flat = [o for _, os_ in e_outs for o in os_]
        for idx, os_ in e_outs:
            for i, o in zip(idx, os_):
                if i in recs:
                    assert o.to_dict() == recs[i], "host and device paths differ"
        return s, flat

    e2e_s, e_flat = e2e_run({})
    full_s, f_flat = e2e_run({"host_crop": 0})
    e2e_value = world * B * K / e2e_s
    h2d_bytes = sum(o.h2d_bytes for o in e_flat) / len(e_flat)

    # ---- rooflines ----
    V = c.vertex_count
    fp32_peak = max(_native.probe_fp32_peak(dev, m) for m in (0, 1, 3))
    fp32_ffma2 = _native.probe_fp32_peak(dev, 0)
    traffic = ncu_traffic()
    mask_bytes = d0.numel()

    def pass1_roof(m, d, label):
        # One fused kernel runs the 3-D list (8 flop per pair: 3 FMA + |p|^2
        # fold + max) and the planar list (6 flop per pair: 2 FMA + fold + max).
        # Pass 1 evaluates the vertices of every kept unit that pass its reach
        # filter: the pair slots it actually evaluates are counted on the
        # device (diagnostics pass1_pairs / pass1_planar_pairs).
        p3 = d["pass1_pairs"]
        p2 = d["pass1_planar_pairs"]
        t = m["pass1_ms"] / 1e3
        ach = (8.0 * p3 + 6.0 * p2) / t / 1e12
        return {"kernel": "diam_pass1", "bound": "fp32", "achieved": ach, "peak": fp32_peak,
                "unit": "TFLOP/s", "frac": ach / fp32_peak,
                "traffic": traffic.get("diam_pass1"),
                "work": f"{label}: 8 flop x {p3:.4g} evaluated 3-D pair slots (vertex-filtered "
                        f"{d['work_subunits']} listed 64x64 sub-pairs of {d['work_units']} kept / "
                        f"{d['total_units']} 128x128 chunk pairs) + 6 flop x {p2:.4g} in-plane "
                        f"pair slots ({d['planar_work_subunits']} listed sub-pairs)",
                "pair_evals_per_s": (p3 + p2) / t,
                "peak_note": "FP32 CUDA-core rate measured on this GPU by sc_probe_fp32_peak "
                             f"(best of FFMA/FFMA-imm/FFMA2; FFMA2 alone {fp32_ffma2:.1f} "
                             "TFLOP/s); nominal 74.4 at 1965 MHz"}

    def pack_roof(ms, kernel, note):
        gbs = mask_bytes / (ms / 1e3) / 1e9
        return {"kernel": kernel, "bound": "hbm", "achieved": gbs, "peak": hbm, "unit": "GB/s",
                "frac": gbs / hbm, "traffic": traffic.get(kernel), "peak_kind": peak_kind,
                "work": f"{mask_bytes} mask bytes read once per launch (one launch per ROI)",
                "mvoxels_per_s": mask_bytes / (ms / 1e3) / 1e6, "timing": note}

    roof_tma = pack_roof(med_tma["pack_ms"], "pack_bits_tma",
                         "CUDA events around the kernel in a single call (option "
                         "pack_tma_single=1, fused bbox), the batch path's pack")
    # The same kernel as the batch runs it: a B-ROI device batch with only
    # init_stats + pack_bits_tma enqueued per ROI (option debug_stages=2:
    # timing only, results discarded), CUDA events on the caller's stream
    # around the batch; launch duration = batch time / B (the pack chain keeps
    # 4 packs in flight, so this is the per-launch share of the HBM stream).
    pk_ms = pack_batch_ms(sc, _native, d_masks, sps, B, stream)
    pk_bytes = sum(roi_bytes[i % len(d_masks)] for i in range(B)) / B
    gbs_b = pk_bytes / (pk_ms / 1e3) / 1e9
    roof_batch = {"kernel": "pack_bits_tma", "bound": "hbm", "achieved": gbs_b, "peak": hbm,
                  "unit": "GB/s", "frac": gbs_b / hbm, "traffic": traffic.get("pack_bits_tma"),
                  "peak_kind": peak_kind,
                  "work": f"{pk_bytes:.4g} mask bytes (mean over the step's ROIs) read once per "
                          "launch, one launch per ROI",
                  "launch_us": pk_ms * 1e3,
                  "timing": "in the batch: B ROIs of init_stats + pack_bits_tma only "
                            "(debug_stages=2), CUDA events around the batch / B",
                  "single_launch": {"achieved": roof_tma["achieved"],
                                    "frac": roof_tma["frac"], "timing": roof_tma["timing"]}}
    roof_v16 = pack_roof(med["pack_ms"], "pack_bits_v16",
                         "CUDA events around the kernel in a single call (128-bit-load pack, "
                         "the single-call path)")
    roof_mc = dict(roof_v16)
    roof_mc["mc_stage_mvoxels_per_s"] = mask_bytes / ((med["pack_ms"] + med["mc_ms"]) / 1e3) / 1e6
    roof_mc["mc_stage_frac_hbm"] = (mask_bytes / ((med["pack_ms"] + med["mc_ms"]) / 1e3) / 1e9
                                    / hbm)
    roof_p1 = pass1_roof(med, diag, "pruned")
    roof_p1_bf = pass1_roof(bf_med, bf_diag, "all pairs")
    stage = {k: v for k, v in med.items() if k != "h2d_ms"}
    dominant = max(stage, key=stage.get)
    # The batch path's dominant kernel is the HBM stream unless pass 1 is the
    # largest single-call stage (C3-like meshes).
    roofline = roof_p1 if dominant == "pass1_ms" else roof_batch
    total_k = sum(stage.values())
    # The largest single kernel of this workload's one-ROI call (the stage
    # groups prune_ms / planar_prep_ms are 3-6 latency-bound kernels each and
    # are reported as groups in kernel_share): its time, share and bound, with
    # the committed ncu counters of that kernel where a capture exists.
    kname = {"pack_ms": "pack_bits_v16", "mc_ms": "mc_cells", "pass1_ms": "diam_pass1",
             "refine_ms": "diam_refine"}
    single = {k: stage[k] for k in kname if k in stage}
    dk = max(single, key=single.get)
    kbound = {"pack_ms": "HBM (roofline_pack_single)",
              "mc_ms": "ALU issue + L2 latency: integer bit ops on the L2-resident bit volume "
                       "(no HBM or FMA roofline applies; see issue_pct)",
              "pass1_ms": "FP32 FMA pipe after pruning: per-unit overhead (roofline_pass1)",
              "refine_ms": "FP64 / latency: re-check of the candidate units"}[dk]
    dom_k = {"kernel": kname[dk], "us": single[dk] * 1e3, "share_of_call": single[dk] / total_k,
             "bound": kbound, "largest_group": max(stage, key=stage.get),
             "largest_group_share": max(stage.values()) / total_k}
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as fh:
            kc = json.load(fh).get("kernels", {}).get(kname[dk])
        if kc:
            dom_k["ncu_c2_capture"] = {k: kc[k] for k in ("issue_pct", "occupancy_pct",
                                                          "pipe_alu_pct", "pipe_fma_pct",
                                                          "dram_pct") if k in kc}
    except (OSError, ValueError):
        pass

    line = {
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": world,
        "steps": K,
        "warmup": W,
        "ms_per_step": dev_ms / K,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "u8 mask; exact int64 MC sums; fp32 screen + fp64 exact diameters",
        "data": "synthetic",
        "config": {"workload": WORKLOADS[args.workload], "name": args.workload,
                   "global_batch": B * world, "rois_per_step_per_gpu": B,
                   "distinct_rois_per_rank": len(d_masks),
                   "roi_bytes_mean": step_bytes,
                   "l2": "no flush: every mask (>= 100 MB) streams from HBM; consecutive ROIs "
                         "of a step are distinct masks" if args.workload == "c4" else
                         ("no flush: the mask (> 126 MB L2) streams from HBM every ROI"
                          if mask_bytes > 126e6 else "mask < L2 (re-read from L2)"),
                   "parallelism": f"roi-batch x{world} (LPT shares, no collective)"},
        "path": "sc_calculate_coefficients_device_batch (C ABI), device-resident masks, one "
                "call of B ROIs per step",
        "roi_ceiling": ceiling(us_roi, step_bytes),
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d_bytes * B),
                # per ROI the last kernel publishes the merged record (2,504 B: the
                # summed case histogram + the tail of sc::Stats) to mapped pinned memory
                "d2h_bytes_per_step": 2504 * B,
                "path": "sc_calculate_coefficients_batch (C ABI) from pinned host memory, B ROIs "
                        "per step: host scan of every mask byte for the occupied z/y slab "
                        "(host_threads), then only that slab crosses PCIe",
                "distinct_host_masks": n_host,
                "mask_bytes_per_step": int(sum(h_masks[i % n_host].size for i in range(B))),
                "host_threads_per_rank": min(32, host_threads),
                "host_scan_ms_per_roi": statistics.median(o.host_scan_ms for o in e_flat),
                "full_copy": {"value": world * B * K / full_s, "unit": UNIT,
                              "h2d_bytes_per_step": int(sum(o.h2d_bytes for o in f_flat)
                                                        / len(f_flat) * B),
                              "note": "option host_crop=0: every mask byte crosses PCIe"}},
        "single_roi": {"value": world * 1e3 / statistics.median(single_ms), "unit": UNIT,
                       "path": "sc_calculate_coefficients_device, one synchronous call per ROI "
                               "(host wall time, median)"},
        "gpu_launches": int(launches),
        "roofline": roofline,
        "roofline_pack_single": roof_mc,
        "roofline_pass1": roof_p1,
        "allpairs": {"value": world * 1e3 / sum(bf_med.values()), "unit": UNIT,
                     "note": "same exact results with pruning disabled (every pair evaluated); "
                             "value from the summed stage times",
                     "kernel_ms": bf_med, "roofline_pass1": roof_p1_bf},
        "kernel_ms": med,
        "kernel_ms_batch_pack": {"pack_ms": med_tma["pack_ms"]},
        "kernel_share": {k: v / total_k for k, v in stage.items()},
        "dominant_stage": dominant,
        "dominant_kernel": dom_k,
        "diagnostics": diag,
        "clocks": clocks.summary(),
        "result": {"VertexCount": V, "triangles": c.triangle_count, "active_cubes": c.active_cubes,
                   "Maximum3DDiameter": c.max_3d_diameter, "MeshVolume": c.mesh_volume,
                   "pairs": V * (V - 1) / 2},
    }
    if side is not None:
        line["c2"] = side
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_sample(gens, args.cpu_seconds / 5, 3)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    return 0


def run_split(args):
    """one very large ROI, its pair grid split across the ranks.
    Every rank runs marching cubes (cheap) and its 1/N of the surviving 3-D and
    planar work units; the 4 squared maxima are combined with one NCCL
    all_reduce(MAX).  Time per step = max over ranks; "scaling": "strong"."""
    import torch

    import paper_2510_02894_b200 as sc
    from paper_2510_02894_b200 import sharding

    world, rank, local = dist_setup(args.gpus)
    dev = torch.cuda.current_device()
    rois, cfg = load_workload(args.workload, 0, 1)
    mask, sp = rois[0]
    d_mask = torch.from_numpy(mask).to(f"cuda:{dev}")
    if args.sim_shards:
        return run_split_sim(args, d_mask, sp, cfg)
    split = (sharding.slab_sharded_coefficients if args.split_mode == "slab"
             else sharding.sharded_coefficients)
    for _ in range(max(3, args.warmup)):
        rec = split(d_mask, sp)
    torch.cuda.synchronize()
    barrier(world)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(dev)
    clocks.__enter__()
    ev0.record()
    for _ in range(args.steps):
        rec = split(d_mask, sp)
    ev1.record()
    torch.cuda.synchronize()
    clocks.__exit__(None, None, None)
    ms = max_over_ranks(world, ev0.elapsed_time(ev1))
    barrier(world)
    full = sc.calculate_coefficients_device(d_mask, sp)
    for k in ("Maximum3DDiameter", "Maximum2DDiameterXY", "Maximum2DDiameterXZ",
              "Maximum2DDiameterYZ", "VertexCount"):
        assert rec[k] == full.to_dict()[k], k
    cfg.update({"global_batch": 1, "parallelism": (
        f"slab split x{world}: marching cubes by cell layers + NCCL all_reduce(SUM) / all_gather "
        f"of the partials and keys, pair grid by identity + NCCL all_reduce(MAX)"
        if args.split_mode == "slab" else
        f"pair-grid split x{world} + NCCL all_reduce(MAX)")})
    line = {"metric": METRIC, "value": args.steps / (ms / 1e3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "u8 mask; exact int64 MC sums; fp32 screen + fp64 exact diameters",
            "data": "synthetic", "config": cfg, "clocks": clocks.summary(),
            "path": ("sharding.slab_sharded_coefficients -> sc_shard_mesh / sc_shard_diameters"
                     if args.split_mode == "slab" else
                     "sharding.sharded_coefficients -> sc_calculate_coefficients_shard"),
            "result": {k: rec[k] for k in ("VertexCount", "Maximum3DDiameter")}}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    return 0


def run_split_sim(args, d_mask, sp, cfg):
    """1-GPU view of the N-GPU split: every shard's phases run one after
    another here, each timed alone (synchronous calls, host wall clock, median
    of the repeats).  The critical path of an N-GPU run is then max over shards
    of phase 1 + max over shards of phase 2 (+ the exchange, not simulated);
    reported beside the single call and the one-call pair-grid shard entry."""
    import statistics

    import torch

    import paper_2510_02894_b200 as sc
    from paper_2510_02894_b200 import sharding

    def wall(fn, reps):
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            fn()
            ts.append((time.perf_counter() - t0) * 1e3)
        return statistics.median(ts)

    reps = max(3, args.steps)
    for _ in range(max(3, args.warmup)):
        full = sc.calculate_coefficients_device(d_mask, sp)
    single_ms = wall(lambda: sc.calculate_coefficients_device(d_mask, sp), reps)
    out = {}
    for n in args.sim_shards:
        times = {}

        def timer(phase, shard, fn):
            res = [None]

            def call():
                res[0] = fn()
            times.setdefault((phase, shard), []).append(wall(call, 1))
            return res[0]

        for _ in range(max(2, args.warmup)):
            rec = sharding.simulate_slab_shards(d_mask, sp, n)
        times.clear()
        for _ in range(reps):
            rec = sharding.simulate_slab_shards(d_mask, sp, n, timer=timer)
        fd = full.to_dict()
        assert all(rec[k] == fd[k] for k in fd if k in rec and not k.endswith("_ms")), n
        p1 = [statistics.median(times[(1, s)]) for s in range(n)]
        p2 = [statistics.median(times[(2, s)]) for s in range(n)]
        sq = torch.zeros(4, dtype=torch.float64, device=d_mask.device)
        pair_ms = [wall(lambda s=s: sc.calculate_coefficients_shard(d_mask, sp, s, n, sq), reps)
                   for s in range(n)]
        crit = max(p1) + max(p2)
        out[str(n)] = {"phase1_ms": p1, "phase2_ms": p2, "critical_ms": crit,
                       "critical_frac_of_single": crit / single_ms,
                       "pair_grid_entry_ms": pair_ms,
                       "pair_grid_frac_of_single": max(pair_ms) / single_ms}
    line = {"metric": "per-shard critical path of the C3 split, simulated on 1 GPU",
            "unit": "ms", "workload": cfg.get("workload"), "single_call_ms": single_ms,
            "shards": out, "exact": True,
            "note": "phase 1 = sc_shard_mesh (pack + marching cubes on the shard's cell "
                    "layers), phase 2 = sc_shard_diameters (load summed partials + gathered "
                    "keys, shard of the pair grid); exchange (all_reduce SUM + all_gather of "
                    "keys over NVLink) not included; host wall clock of synchronous calls, "
                    f"median of {reps}"}
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=300,
                    help="ROIs per step per GPU (default: the C4 batch size, 300)")
    ap.add_argument("--e2e-masks", type=int, default=16,
                    help="distinct pinned host masks cycled by the e2e leg")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-side", action="store_true", help="skip the C2 side-by-side line")
    ap.add_argument("--cpu-seconds", type=float, default=170.0)
    ap.add_argument("--workload", default="c4", choices=sorted(WORKLOADS))
    ap.add_argument("--split", action="store_true",
                    help="strong scaling of ONE ROI: every rank evaluates its share of the pair "
                         "grid (sc_calculate_coefficients_shard) + one NCCL all_reduce(MAX)")
    ap.add_argument("--split-mode", default="slab", choices=["slab", "pairs"],
                    help="slab: marching cubes split by cell layers too (sc_shard_mesh / "
                         "sc_shard_diameters); pairs: one-call pair-grid shard entry")
    ap.add_argument("--sim-shards", type=int, nargs="*", default=None,
                    help="with --split on 1 GPU: time every shard of an N-way slab split "
                         "(one after another) and report the per-shard critical path")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3  # contract: W >= 3 warm-up steps
    if args.impl == "reference":
        return run_reference(args)
    if args.split:
        return run_split(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
