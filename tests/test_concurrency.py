"""Concurrency and stream-ordering contracts of the C ABI.

* SPEC.md:234 / :386 -- calls are made "concurrently from multiple threads on
  distinct meshes": host threads x distinct masks through the host, device and
  batch entries give exactly the sequential results.
* Options are snapshotted per call: a thread changing its own options
  (sc_set_thread_option) or the process-wide ones never changes another
  thread's in-flight call.
* A device mask written by torch on the caller's stream (default or side
  stream) is read only after that write: the entries order themselves after
  prior work on the stream they are given -- NULL meaning the legacy default
  stream (the library's slot streams are non-blocking).
"""

import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _masks():
    from paper_2510_02894_b200 import synth

    rng = np.random.default_rng(99)
    out = []
    for i in range(8):
        nx, ny, nz = (int(v) for v in rng.integers(24, 72, size=3))
        a = np.zeros((nz, ny, nx), dtype=np.uint8)
        for _ in range(int(rng.integers(1, 5))):
            c = rng.uniform(3, [nz - 3, ny - 3, nx - 3])
            r = rng.uniform(2, 9)
            zz, yy, xx = np.ogrid[:nz, :ny, :nx]
            a |= (((zz - c[0]) ** 2 + (yy - c[1]) ** 2 + (xx - c[2]) ** 2) <= r * r).astype(np.uint8)
        a[nz // 2, ny // 2, nx // 2] = 1
        sp = tuple(float(v) for v in rng.choice([0.5, 0.8, 1.0, 1.25, 3.0], size=3))
        out.append((a, sp))
    out.append((synth.kits_like(256, 256, 200, (0.8, 0.8, 1.0), 30.0), (0.8, 0.8, 1.0)))
    return out


def test_threads_distinct_masks_equal_sequential(sc, cuda_device):
    import torch

    from paper_2510_02894_b200 import _native

    cases = _masks()
    want = [sc.calculate_coefficients(a, sp).to_dict() for a, sp in cases]
    errors = []

    def host_worker(tid):
        try:
            for rep in range(3):
                for i in range(tid % 3, len(cases), 2):
                    a, sp = cases[i]
                    got = sc.calculate_coefficients(a, sp).to_dict()
                    assert got == want[i], (tid, i)
        except Exception as exc:  # noqa: BLE001 - reported below
            errors.append(repr(exc))

    def device_worker(tid):
        try:
            stream = torch.cuda.Stream()
            with torch.cuda.stream(stream):
                ds = [torch.from_numpy(a).cuda() for a, _ in cases]
                for rep in range(3):
                    i = (tid + rep) % len(cases)
                    got = sc.calculate_coefficients_device(ds[i], cases[i][1], stream=stream)
                    assert got.to_dict() == want[i], (tid, i)
                got = sc.calculate_coefficients_device_batch(ds, [sp for _, sp in cases],
                                                             stream=stream)
                assert [g.to_dict() for g in got] == want, tid
        except Exception as exc:  # noqa: BLE001
            errors.append(repr(exc))

    def option_worker(tid):
        # this thread's own options change its own calls only, and the results
        # stay identical (pruning / graphs / launch shape never change a result)
        try:
            with _native.thread_options(prune=0, graphs=0, grid_div_single=3, slots=4):
                for i in range(0, len(cases), 3):
                    a, sp = cases[i]
                    assert sc.calculate_coefficients(a, sp).to_dict() == want[i], (tid, i)
                got = sc.calculate_coefficients_batch([a for a, _ in cases],
                                                      [sp for _, sp in cases])
                assert [g.to_dict() for g in got] == want, tid
        except Exception as exc:  # noqa: BLE001
            errors.append(repr(exc))

    threads = [threading.Thread(target=f, args=(t,))
               for t, f in enumerate([host_worker, host_worker, device_worker, device_worker,
                                      option_worker])]
    for t in threads:
        t.start()
    # meanwhile flip a process-wide option back and forth: in-flight calls keep
    # the snapshot they took at entry, and results never depend on it
    for _ in range(20):
        _native.set_option("fork", 0)
        _native.set_option("fork", 1)
    for t in threads:
        t.join(timeout=600)
    assert not errors, errors


def test_thread_options_are_per_thread(sc, cuda_device):
    """sc_set_thread_option affects only the calling thread; the process-wide
    value is untouched (checked through a value only the option changes)."""
    from paper_2510_02894_b200 import _native, synth

    a = synth.kits_like(256, 256, 200, (0.8, 0.8, 1.0), 30.0)
    # (work_units depends on the host crop's slab origin, total_units only on V)
    sc.calculate_coefficients(a, (0.8, 0.8, 1.0))
    d = _native.last_diagnostics(cuda_device)
    assert d["work_units"] < d["total_units"]  # pruning on
    with _native.thread_options(prune=0):
        sc.calculate_coefficients(a, (0.8, 0.8, 1.0))
        d = _native.last_diagnostics(cuda_device)
        assert d["work_units"] == d["total_units"]  # pruning off for this thread
        seen = {}

        def other():
            sc.calculate_coefficients(a, (0.8, 0.8, 1.0))
            seen.update(_native.last_diagnostics(cuda_device))

        t = threading.Thread(target=other)
        t.start()
        t.join()
    assert seen["work_units"] < seen["total_units"]  # the other thread still prunes
    sc.calculate_coefficients(a, (0.8, 0.8, 1.0))
    d = _native.last_diagnostics(cuda_device)
    assert d["work_units"] < d["total_units"]  # and so does this one afterwards


@pytest.mark.parametrize("side_stream", [False, True])
def test_device_entry_ordered_after_torch_writes(sc, cuda_device, side_stream):
    """The mask is produced by torch behind a ~50 ms spin kernel on the
    caller's (current) stream; the call must see the finished mask."""
    import torch

    from paper_2510_02894_b200 import synth

    a = synth.kits_like(256, 256, 160, (0.8, 0.8, 1.0), 40.0)
    want = sc.calculate_coefficients(a, (0.8, 0.8, 1.0)).to_dict()
    src = torch.from_numpy(a).cuda()
    stream = torch.cuda.Stream() if side_stream else torch.cuda.current_stream()
    torch.cuda.synchronize()
    with torch.cuda.stream(stream):
        for _ in range(3):
            dst = torch.zeros_like(src)
            torch.cuda._sleep(100_000_000)  # ~50 ms of device spin before the write
            dst.copy_(src)
            got = sc.calculate_coefficients_device(dst, (0.8, 0.8, 1.0))  # current stream
            assert got.to_dict() == want
            dst = torch.zeros_like(src)
            torch.cuda._sleep(100_000_000)
            dst.copy_(src)
            outs = sc.calculate_coefficients_device_batch([dst, dst], [(0.8, 0.8, 1.0)] * 2)
            assert [o.to_dict() for o in outs] == [want, want]
    torch.cuda.synchronize()


def test_null_stream_means_legacy_default_stream(sc, cuda_device):
    """C level: stream = NULL orders the call after work on the legacy default
    stream (torch's default stream is that stream)."""
    import ctypes

    import torch

    from paper_2510_02894_b200 import _native, synth

    a = synth.kits_like(256, 256, 160, (0.8, 0.8, 1.0), 40.0)
    want = sc.calculate_coefficients(a, (0.8, 0.8, 1.0)).to_dict()
    src = torch.from_numpy(a).cuda()
    sp = np.asarray((0.8, 0.8, 1.0), dtype=np.float64)
    torch.cuda.synchronize()
    with torch.cuda.stream(torch.cuda.default_stream()):
        dst = torch.zeros_like(src)
        torch.cuda._sleep(100_000_000)
        dst.copy_(src)
        nz, ny, nx = dst.shape
        out = _native.ScCoeffs()
        rc = _native.load().sc_calculate_coefficients_device(
            ctypes.c_void_p(dst.data_ptr()), nx, ny, nz,
            sp.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), ctypes.c_void_p(0),
            ctypes.byref(out))
        assert rc == 0
    from paper_2510_02894_b200.features import _from_struct

    assert _from_struct(out).to_dict() == want


def test_batch_multi_fans_out_in_input_order(sc, cuda_device):
    """sc_calculate_coefficients_batch_multi: LPT fan-out over a device list
    inside the C ABI; on one GPU the list repeats device 0 (two / three host
    worker threads sharing it) -- records equal the single-device batch, in
    input order, and an input error in one ROI leaves the others computed."""
    from paper_2510_02894_b200 import errors

    cases = _masks()
    masks, sps = [a for a, _ in cases], [sp for _, sp in cases]
    want = [c.to_dict() for c in sc.calculate_coefficients_batch(masks, sps)]
    for devs in ([0], [0, 0], [0, 0, 0]):
        got = sc.calculate_coefficients_batch(masks, sps, devices=devs)
        assert [g.to_dict() for g in got] == want, devs
    bad = list(sps)
    bad[3] = (1.0, -1.0, 1.0)
    with pytest.raises(errors.ShapeCoreError):
        sc.calculate_coefficients_batch(masks, bad, devices=[0, 0])
    with pytest.raises((ValueError, errors.ShapeCoreError)):
        sc.calculate_coefficients_batch(masks, sps, devices=[0, 57])  # no such device
