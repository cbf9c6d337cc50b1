"""Benchmark: ROIs/s of full 3-D shape coefficients on KiTS19-shaped masks.

Contract (driver): `python bench.py --gpus N --steps K --warmup W` prints ONE
JSON line on rank 0.  N>1 runs under torchrun, one rank per GPU; every rank
processes its own ROIs (ROI-batch sharding: independent masks, no data-path
collective -> "scaling": "weak"); the timed region is bracketed by a barrier
and torch.cuda.synchronize() and the reported time is the max over ranks.

Workload (BASELINE.json configs[1]): one synthetic KiTS19-shaped mask,
512x512x600 uint8 at 0.8x0.8x1.0 mm, two kidneys + a 30 mm tumour
(SURVEY.md Appendix D, V = 73,406 vertices).  One step = calculate_coefficients
of one ROI: marching cubes -> area/volume -> 3-D and planar diameters.  The
mask (157 MB) is larger than L2 (126 MB), so no L2 flush is needed.

  value      device-resident throughput: mask already in HBM, K ROIs through the
             pipelined device batch entry, CUDA events on the caller's stream
             (the batch is ordered against it), host round trips included.
  e2e        the same metric through the C ABI with a HOST (pinned) mask: the
             pipelined host batch entry copies the 157 MB mask H2D for every
             ROI and reads every result back.
  single_roi one synchronous call per ROI (no cross-ROI overlap); its
             per-kernel CUDA-event times feed kernel_ms and the rooflines.
  roofline   the dominant kernel of the step.  diam3d_pass1 is FP32
             CUDA-core bound: achieved = 8 flop x evaluated pairs / kernel time,
             peak = FP32 rate measured by sc_probe_fp32_peak on this GPU.
             pack_bits_v16 is HBM-bound: achieved = mask bytes / kernel time vs
             the measured copy bandwidth in MEASURED_PEAKS.json.
  allpairs   the same exact results with work pruning disabled (every pair
             through pass 1): the brute-force pass-1 roofline.
  cpu_baseline  the CPU oracle (C restatement of the reference, OpenMP strip-
             parallel diameters, serial MC as in the reference) on one ROI.

`--impl reference` times that CPU path alone (rank 0; other ranks exit 0).
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

# SURVEY.md 8(d) configurations.  The default (headline, BASELINE.json
# configs[1]) is c2; the others are selectable with --workload.
WORKLOADS = {
    "c1": "C1 synthetic 64^3 sphere mask (r=24, spacing 1 mm, V=10824; the reference's own "
          "CPU-runnable case), one ROI per step per GPU",
    "c2": "C2 KiTS19-shaped synthetic kidney+tumor mask 512x512x600 uint8 at 0.8x0.8x1.0 mm "
          "(tumor 30 mm, V=73406), one ROI per step per GPU",
    "c3": "C3 noisy-boundary ellipsoid 512^3 at 1 mm (sigma 0.02, seed 1234, V=1963474, "
          "1.93e12 pairs), one ROI per step per GPU",
    "c4": "C4 batch of 300 varied KiTS19-shaped masks (512x512x[200..700], seed 2025), "
          "LPT-sharded across GPUs, one ROI per step, cycling the rank's share",
    "c5": "C5 thin slab 512x512x24 at 0.5x0.5x5 mm, 400 blobs (seed 7, V=127664), "
          "one ROI per step per GPU",
}


def load_workload(name, rank=0, world=1):
    """[(mask (nz,ny,nx) uint8, spacing)] for this rank, plus a config dict."""
    from paper_2510_02894_b200 import sharding, synth

    if name == "c1":
        rois = [(synth.synth_mask("sphere", (64, 64, 64), radius=24), (1.0, 1.0, 1.0))]
    elif name == "c2":
        rois = [(synth.kits_like(512, 512, 600, (0.8, 0.8, 1.0), 30.0), (0.8, 0.8, 1.0))]
    elif name == "c3":
        rois = [(synth.noisy_ellipsoid(512, 0.02, 1234), (1.0, 1.0, 1.0))]
    elif name == "c5":
        rois = [(synth.thin_slab(), (0.5, 0.5, 5.0))]
    elif name == "c4":
        params = synth.kits_batch_params(300, 2025)
        # cost: streamed voxels + (surface ~ tumour/kidney size)^2 pairs
        costs = [sharding.roi_cost(int((p["tumor_mm"] / p["sp"][0]) ** 3 * 4.2 + 2.6e5),
                                   p["nx"] * p["ny"] * p["nz"]) for p in params]
        mine = sharding.assign_rois(costs, world)[rank]
        rois = [(synth.kits_from_params(params[i]), tuple(params[i]["sp"])) for i in mine]
    else:
        raise SystemExit(f"unknown workload {name}")
    cfg = {
        "workload": WORKLOADS[name],
        "name": name,
        "global_batch": None,
        "roi_bytes_mean": sum(m.size for m, _ in rois) / max(1, len(rois)),
        "rois_per_rank": len(rois),
        "l2": "every mask > 126 MB L2 (no flush needed)" if min(m.size for m, _ in rois) > 126e6
              else "mask < L2: steps cycle distinct ROIs / the mask is re-read from L2",
        "parallelism": None,
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


def cpu_reference_time(mask, spacing, max_seconds=150.0, steps=1, warmup=0):
    """The oracle (C port of the reference path) on all host cores: MC serial
    (mesh.py:68-199), diameters strip-parallel (features.py:151-192).
    Returns (per-ROI seconds list, threads, sample description).  When the
    full pair loop would exceed the budget (C3), the diameters are timed on a
    random vertex subset and extrapolated by pair count (labelled as such)."""
    import numpy as np

    from oracle import oracle

    threads = oracle.max_threads()
    t0 = time.perf_counter()
    mesh = oracle.marching_cubes(mask, spacing)
    t_mc = time.perf_counter() - t0
    V = mesh.vertex_count
    pairs = V * (V - 1) / 2
    if pairs <= 4e10:
        t_start = time.perf_counter()
        for _ in range(warmup):
            oracle.extract_features(mask, spacing, threads=0, with_active=False)
            if time.perf_counter() - t_start > max_seconds / 2:
                break
        times = []
        for _ in range(max(1, steps)):
            t1 = time.perf_counter()
            oracle.extract_features(mask, spacing, threads=0, with_active=False)
            times.append(time.perf_counter() - t1)
            if time.perf_counter() - t_start > max_seconds:
                break
        return times, threads, f"{len(times)} full ROI(s)"
    m = int((2 * 2e10) ** 0.5)
    idx = np.sort(np.random.default_rng(0).choice(V, size=m, replace=False))
    t1 = time.perf_counter()
    oracle.diameters(mesh.xs[idx], mesh.ys[idx], mesh.zs[idx], threads=0)
    t_d = (time.perf_counter() - t1) * pairs / (m * (m - 1) / 2)
    t_area = 0.0
    t2 = time.perf_counter()
    oracle.surface_area(mesh)
    oracle.mesh_volume(mesh)
    t_area = time.perf_counter() - t2
    return [t_mc + t_area + t_d], threads, (
        f"full MC ({t_mc:.1f}s) + area/volume + diameters timed on a {m}-vertex random subset "
        f"and extrapolated by pair count ({pairs:.3g} pairs -> {t_d:.0f}s)")


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return 0
    rois, cfg = load_workload(args.workload, 0, 1)
    mask, sp = rois[len(rois) // 2]
    times, threads, sample = cpu_reference_time(mask, sp, max_seconds=args.cpu_seconds,
                                                steps=args.steps, warmup=min(args.warmup, 1))
    per = statistics.mean(times)
    value = 1.0 / per
    cfg.update({"parallelism": "host cores (OpenMP)", "global_batch": 1})
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference",
        "n_gpus": world, "steps": len(times), "warmup": min(args.warmup, 1),
        "ms_per_step": per * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u8/fp64", "data": "synthetic",
        "config": cfg,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{sample} through oracle/shape_oracle.c (reference "
                                   "algorithm restated in C: serial canonical MC, "
                                   "strip-parallel fp64 diameters), time-capped at "
                                   f"{args.cpu_seconds:.0f}s"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def measure_device(sc, _native, d_mask, sp, stream, steps, warmup, dev, world):
    """One synchronous call per ROI (no cross-ROI overlap): K steps on `stream`,
    CUDA events around the loop (default graph events: mesh / diameters only);
    then the same number of calls with an event at every stage boundary
    (option stage_times=2) for the per-kernel medians.  Returns (ms max over
    ranks, per-kernel median ms, diagnostics, launches, last result)."""
    import torch

    with torch.cuda.stream(stream):
        for _ in range(warmup):
            c = sc.calculate_coefficients_device(d_mask, sp, stream=stream)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = _native.launch_count()
    barrier(world)
    torch.cuda.synchronize()
    ev0.record(stream)
    for _ in range(steps):
        c = sc.calculate_coefficients_device(d_mask, sp, stream=stream)
    ev1.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    launches = _native.launch_count() - launches0
    ms = max_over_ranks(world, ev0.elapsed_time(ev1))
    kt = {k: [] for k in _native.KERNEL_TIME_NAMES}
    _native.set_option("stage_times", 2)
    try:
        sc.calculate_coefficients_device(d_mask, sp, stream=stream)  # captures its graph
        for _ in range(steps):
            sc.calculate_coefficients_device(d_mask, sp, stream=stream)
            for k, v in _native.last_kernel_times(dev).items():
                kt[k].append(v)
    finally:
        _native.set_option("stage_times", 0)
    med = {k: statistics.median(v) for k, v in kt.items() if v}
    return ms, med, _native.last_diagnostics(dev), launches, c


def run_ours(args):
    import numpy as np
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
    rois, cfg = load_workload(args.workload, rank, world)
    d_masks = [torch.from_numpy(m).to(f"cuda:{dev}") for m, _ in rois]
    sps = [sp for _, sp in rois]
    stream = torch.cuda.Stream()
    n_host = min(len(rois), 8)
    h_masks = [torch.from_numpy(m).pin_memory().numpy() for m, _ in rois[:n_host]]
    K = args.steps
    step_masks = [d_masks[i % len(d_masks)] for i in range(K)]
    step_sps = [sps[i % len(sps)] for i in range(K)]

    # ---- device-resident throughput (value): K ROIs through the pipelined
    # device batch entry (16 slots: ROI i+16 is enqueued when ROI i is
    # collected), CUDA events on `stream`, which the batch is ordered against.
    clocks = ClockSampler(dev)
    W = args.warmup
    # W warm-up steps, and at least two rounds over the 16 pipeline slots so
    # every slot has captured its CUDA graph before the timed region.
    # Then one untimed batch of exactly the timed shape: the first K-ROI batch
    # after the capture-bound warm-up (the GPU mostly waits on host-side graph
    # captures there) runs ~15 % slower on the device (C2, K = 20: 57.7 vs 49-50
    # us/ROI for the next ones; host-side launch and collect times identical,
    # tools/k20_probe.py), a one-off a steady stream of batches does not pay.
    Ww = max(W, 32)
    sc.calculate_coefficients_device_batch([d_masks[i % len(d_masks)] for i in range(Ww)],
                                           [sps[i % len(sps)] for i in range(Ww)], stream=stream)
    sc.calculate_coefficients_device_batch(step_masks, step_sps, stream=stream)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = _native.launch_count()
    barrier(world)
    torch.cuda.synchronize()
    clocks.__enter__()
    ev0.record(stream)
    outs = sc.calculate_coefficients_device_batch(step_masks, step_sps, stream=stream)
    ev1.record(stream)
    torch.cuda.synchronize()
    clocks.__exit__(None, None, None)
    barrier(world)
    launches = _native.launch_count() - launches0
    dev_ms = max_over_ranks(world, ev0.elapsed_time(ev1))
    value = world * K / (dev_ms / 1e3)
    for i, o in enumerate(outs[len(d_masks):]):
        assert o.to_dict() == outs[i % len(d_masks)].to_dict()

    # ---- one ROI per call on the first ROI: per-kernel times ----
    d0, sp0 = d_masks[0], sps[0]
    one_steps = max(3, min(K, 30))
    one_ms, med, diag, _, c = measure_device(sc, _native, d0, sp0, stream, one_steps, 3, dev, world)
    assert c.to_dict() == outs[0].to_dict()

    # ---- same, all pairs evaluated (no pruning): the pass-1 roofline case ----
    _native.set_option("prune", 0)
    bf_steps = 3 if args.workload == "c3" else max(3, one_steps // 2)
    bf_ms, bf_med, bf_diag, _, c_bf = measure_device(sc, _native, d0, sp0, stream, bf_steps, 1,
                                                     dev, world)
    _native.set_option("prune", 1)
    assert c_bf.to_dict() == c.to_dict(), "pruned and all-pairs results differ"

    # ---- end to end through the C ABI from pinned host memory (e2e): the
    # pipelined host batch entry; every step copies its mask H2D.
    sc.calculate_coefficients_batch([h_masks[i % n_host] for i in range(16)],
                                    [sps[i % n_host] for i in range(16)], device=dev)
    barrier(world)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e_outs = sc.calculate_coefficients_batch([h_masks[i % n_host] for i in range(K)],
                                             [sps[i % n_host] for i in range(K)], device=dev)
    torch.cuda.synchronize()
    e2e_s = max_over_ranks(world, time.perf_counter() - t0)
    barrier(world)
    e2e_value = world * K / e2e_s
    h2d_bytes = sum(o.h2d_bytes for o in e_outs) / K
    scan_ms = statistics.median(o.host_scan_ms for o in e_outs)
    assert e_outs[0].to_dict() == outs[0].to_dict()
    # same, copying every mask byte (option host_crop off): the PCIe-bound figure
    _native.set_option("host_crop", 0)
    sc.calculate_coefficients_batch([h_masks[i % n_host] for i in range(8)],
                                    [sps[i % n_host] for i in range(8)], device=dev)
    barrier(world)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    f_outs = sc.calculate_coefficients_batch([h_masks[i % n_host] for i in range(K)],
                                             [sps[i % n_host] for i in range(K)], device=dev)
    torch.cuda.synchronize()
    full_s = max_over_ranks(world, time.perf_counter() - t0)
    barrier(world)
    _native.set_option("host_crop", 1)
    assert f_outs[0].to_dict() == outs[0].to_dict()

    # ---- rooflines ----
    V = c.vertex_count
    pairs_alg = V * (V - 1) / 2
    fp32_peak = max(_native.probe_fp32_peak(dev, m) for m in (0, 1, 3))
    fp32_ffma2 = _native.probe_fp32_peak(dev, 0)
    # the committed ncu capture (tools/gpu_final.sh) is of the C2 workload
    traffic = ncu_traffic() if args.workload == "c2" else {}
    peaks, peak_kind = measured_peaks()
    mask_bytes = d0.numel()

    def pass1_roof(m, d, label):
        # One fused kernel runs the 3-D list (8 flop per pair: 3 FMA + |p|^2
        # fold + max) and the planar list (6 flop per pair: 2 FMA + fold + max).
        # Pass 1 evaluates the listed 64 x 64 sub-pairs of every kept unit.
        edge = 64
        sub = _native.PAIRS_PER_UNIT // 4
        p3 = d["work_subunits"] * sub
        p2 = d["planar_work_subunits"] * sub
        t = m["pass1_ms"] / 1e3
        ach = (8.0 * p3 + 6.0 * p2) / t / 1e12
        return {"kernel": "diam_pass1", "bound": "fp32", "achieved": ach, "peak": fp32_peak,
                "unit": "TFLOP/s", "frac": ach / fp32_peak,
                "traffic": traffic.get("diam_pass1"),
                "work": f"{label}: 8 flop x {p3:.4g} 3-D pairs ({d['work_subunits']} {edge}x{edge} "
                        f"sub-pairs of {d['work_units']} kept / {d['total_units']} 128x128 "
                        f"chunk pairs) + 6 flop x {p2:.4g} in-plane pairs "
                        f"({d['planar_work_subunits']} sub-pairs)",
                "pair_evals_per_s": (p3 + p2) / t,
                "peak_note": "FP32 CUDA-core rate measured on this GPU by sc_probe_fp32_peak "
                             f"(best of FFMA/FFMA-imm/FFMA2; FFMA2 alone {fp32_ffma2:.1f} "
                             "TFLOP/s); nominal 74.4 at 1965 MHz"}

    pack_s = med["pack_ms"] / 1e3
    mc_gbs = mask_bytes / pack_s / 1e9
    roof_mc = {"kernel": "pack_bits_v16", "bound": "hbm", "achieved": mc_gbs,
               "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": mc_gbs / peaks["hbm_gbs"],
               "traffic": traffic.get("pack_bits_v16"), "peak_kind": peak_kind,
               "work": f"{mask_bytes} mask bytes read once per launch",
               "mvoxels_per_s": mask_bytes / pack_s / 1e6,
               "mc_stage_mvoxels_per_s": mask_bytes / ((med["pack_ms"] + med["mc_ms"]) / 1e3) / 1e6}
    roof_p1 = pass1_roof(med, diag, "pruned")
    roof_p1_bf = pass1_roof(bf_med, bf_diag, "all pairs")
    stage = {k: v for k, v in med.items() if k != "h2d_ms"}
    dominant = max(stage, key=stage.get)
    roofline = roof_p1 if dominant == "pass1_ms" else roof_mc
    total_k = sum(stage.values())
    cfg.update({"global_batch": world, "parallelism": f"roi-batch x{world}"})

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
        "dtype": "fp32",
        "data": "synthetic",
        "config": cfg,
        "path": "sc_calculate_coefficients_device_batch (C ABI), device-resident masks",
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d_bytes),
                "d2h_bytes_per_step": 16800,  # one Stats record (sizeof(sc::Stats), 8 histogram copies)
                "path": "sc_calculate_coefficients_batch (C ABI, pipelined) from pinned host "
                        "memory: host scan of every mask byte for the occupied z/y slab "
                        "(host_threads), then only that slab is copied H2D",
                "mask_bytes_per_step": int(sum(h_masks[i % n_host].size for i in range(K)) / K),
                "host_threads_per_rank": min(32, host_threads),
                "host_scan_ms_per_roi": scan_ms,
                "h2d_ms_per_roi": e_outs[-1].h2d_ms,
                "full_copy": {"value": world * K / full_s, "unit": UNIT,
                              "h2d_bytes_per_step": int(sum(o.h2d_bytes for o in f_outs) / K),
                              "note": "option host_crop=0: every mask byte crosses PCIe"}},
        "single_roi": {"value": world * one_steps / (one_ms / 1e3), "unit": UNIT,
                       "path": "sc_calculate_coefficients_device, one synchronous call per ROI"},
        "gpu_launches": int(launches),
        "roofline": roofline,
        "roofline_mc": roof_mc,
        "roofline_pass1": roof_p1,
        "allpairs": {"value": world * bf_steps / (bf_ms / 1e3), "unit": UNIT,
                     "note": "same exact results with pruning disabled (every pair evaluated)",
                     "kernel_ms": bf_med, "roofline_pass1": roof_p1_bf},
        "kernel_ms": med,
        "kernel_share": {k: v / total_k for k, v in stage.items()},
        "dominant_stage": dominant,
        "diagnostics": diag,
        "clocks": clocks.summary(),
        "result": {"VertexCount": V, "triangles": c.triangle_count, "active_cubes": c.active_cubes,
                   "Maximum3DDiameter": c.max_3d_diameter, "MeshVolume": c.mesh_volume,
                   "pairs": pairs_alg},
    }

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        m, sp = rois[0]
        times, threads, sample = cpu_reference_time(m, sp, max_seconds=args.cpu_seconds, steps=1)
        per = statistics.mean(times)
        line["cpu_baseline"] = {
            "value": 1.0 / per, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{sample} through oracle/shape_oracle.c (reference algorithm in C: "
                      "serial canonical MC + strip-parallel fp64 diameters on all host threads)",
            "seconds_per_roi": per,
        }
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
    for _ in range(max(3, args.warmup)):
        rec = sharding.sharded_coefficients(d_mask, sp)
    torch.cuda.synchronize()
    barrier(world)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(dev)
    clocks.__enter__()
    ev0.record()
    for _ in range(args.steps):
        rec = sharding.sharded_coefficients(d_mask, sp)
    ev1.record()
    torch.cuda.synchronize()
    clocks.__exit__(None, None, None)
    ms = max_over_ranks(world, ev0.elapsed_time(ev1))
    barrier(world)
    full = sc.calculate_coefficients_device(d_mask, sp)
    for k in ("Maximum3DDiameter", "Maximum2DDiameterXY", "Maximum2DDiameterXZ",
              "Maximum2DDiameterYZ", "VertexCount"):
        assert rec[k] == full.to_dict()[k], k
    cfg.update({"global_batch": 1, "parallelism": f"pair-grid split x{world} + NCCL all_reduce(MAX)"})
    line = {"metric": METRIC, "value": args.steps / (ms / 1e3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "fp32",
            "data": "synthetic", "config": cfg, "clocks": clocks.summary(),
            "path": "sharding.sharded_coefficients -> sc_calculate_coefficients_shard",
            "result": {k: rec[k] for k in ("VertexCount", "Maximum3DDiameter")}}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=150.0)
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--split", action="store_true",
                    help="strong scaling of ONE ROI: every rank evaluates its share of the pair "
                         "grid (sc_calculate_coefficients_shard) + one NCCL all_reduce(MAX)")
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
