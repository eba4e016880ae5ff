"""The reference's concurrency contract on the device handles.

SPEC.md:362,445: the HBS operator and the ELS solver are immutable after
build and concurrent solves with distinct right-hand sides are allowed.
sbx.h promises the same for calls on distinct streams: each stream gets its
own sweep workspace, completion counters and staging (PerStream scratch),
lazy plan builds happen once under the handle's lock, and the persistent
dataflow sweep is a cooperative launch (co-resident grid), so two sweeps in
flight on one handle neither corrupt each other nor deadlock.

Also: an error raised inside compress_update while its A_pp build thread is
running comes back as the reference's exception class, and the library is
still usable afterwards (update.cpp join-on-exit, idengine.cpp rendezvous).
"""
import os
import subprocess
import sys
import threading
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]


@pytest.fixture(scope="module")
def sb():
    import paper_2108_07205_b200 as sb
    sb.init(0)
    return sb


def _run_threads(fns):
    errs = []

    def wrap(f):
        try:
            f()
        except BaseException as e:  # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=wrap, args=(f,)) for f in fns]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not any(t.is_alive() for t in th), "concurrent solves did not finish"
    if errs:
        raise errs[0]


@pytest.mark.parametrize("nrhs", [1, 40])
def test_concurrent_hbs_solves_on_two_streams(sb, nrhs):
    import torch
    g = sb.panelize(sb.star(5, 0.3), 512, 16)  # 16384 unknowns: the sweeps overlap on the chip
    h = sb.hbs_invert(sb.hbs_compress(g))
    n = h.n
    rng = np.random.default_rng(nrhs)
    B = [torch.from_numpy(rng.uniform(-1, 1, (n, nrhs))).cuda() for _ in range(2)]
    # a fresh handle: the first calls race to build the plan and flow items
    ref = []
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    out = [[None] * 12, [None] * 12]

    def worker(i):
        def f():
            with torch.cuda.stream(streams[i]):
                for r in range(12):
                    x = sb.hbs_solve(h, B[i]) if r % 3 else sb.hbs_solve(h, B[i], transpose=True)
                    out[i][r] = x
                streams[i].synchronize()
        return f

    _run_threads([worker(0), worker(1)])
    torch.cuda.synchronize()
    for i in range(2):
        ref = sb.hbs_solve(h, B[i]).cpu().numpy()
        ref_t = sb.hbs_solve(h, B[i], transpose=True).cpu().numpy()
        for r in range(12):
            exp = ref if r % 3 else ref_t
            assert np.array_equal(out[i][r].cpu().numpy(), exp), (i, r)


def test_concurrent_els_solves_on_two_streams(sb):
    import torch
    g0 = sb.panelize(sb.star(5, 0.3), 256, 16)
    h = sb.hbs_invert(sb.hbs_compress(g0))
    g1, plan = sb.refine(g0, [10, 11, 12, 13], 16)  # 2 N_p = 2048: dense A_pp; u columns through a_oo
    u = sb.compress_update(g0, g1, plan, 1e-10)
    e = sb.els_build(h, g0, g1, plan, u)
    rows = e.info()["n_k"] + e.info()["n_p"]
    rng = np.random.default_rng(7)
    G = [torch.from_numpy(rng.standard_normal((rows, w))).cuda() for w in (1, 33)]
    serial = [sb.els_solve(e, Gi).cpu().numpy() for Gi in G]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    out = [[], []]

    def worker(i):
        def f():
            with torch.cuda.stream(streams[i]):
                for _ in range(10):
                    out[i].append(sb.els_solve(e, G[i]))
                streams[i].synchronize()
        return f

    _run_threads([worker(0), worker(1)])
    for i in range(2):
        for x in out[i]:
            assert np.array_equal(x.cpu().numpy(), serial[i])


def test_concurrent_host_pointer_solves(sb):
    """Host buffers through the C-ABI from two threads (library staging per
    stream): both see their own results."""
    import torch
    from paper_2108_07205_b200 import _sbx
    g = sb.panelize(sb.circle(), 64, 16)
    h = sb.hbs_invert(sb.hbs_compress(g))
    n = h.n
    rng = np.random.default_rng(1)
    B = [np.asfortranarray(rng.standard_normal((n, 5))) for _ in range(2)]
    ref = [sb.hbs_solve(h, b) for b in B]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    out = [[], []]

    def worker(i):
        def f():
            for _ in range(20):
                x = np.zeros_like(B[i], order="F")
                _sbx.check(_sbx.lib().sbx_hbs_solve(h.ptr, _sbx.VP(B[i].ctypes.data), n, 5,
                                                    _sbx.VP(x.ctypes.data), n, 0,
                                                    _sbx.VP(streams[i].cuda_stream)))
                out[i].append(x)
        return f

    _run_threads([worker(0), worker(1)])
    for i in range(2):
        for x in out[i]:
            assert np.array_equal(x, ref[i])


def test_update_error_with_app_thread_running_is_reported(tmp_path):
    """A ProxyViolation raised by the update's main thread while the A_pp
    HBS build runs in its worker thread (SBX_PAR_MODE 4) unwinds cleanly:
    status 5 through the C-ABI, no terminate(), library usable afterwards."""
    code = r"""
import numpy as np, paper_2108_07205_b200 as sb
sb.init(0)
g0 = sb.panelize(sb.star(5, 0.3), 256, 16)
h = sb.hbs_invert(sb.hbs_compress(g0))
g1, plan = sb.refine(g0, list(range(10, 18)), 16)   # 2 N_p = 4096: A_pp HBS in the worker thread
for _ in range(3):
    try:
        sb.compress_update(g0, g1, plan, 1e-10)
    except sb.ProxyViolationError as e:
        assert "SBX_TEST_FAULT" in str(e)
    else:
        raise SystemExit("no error")
b = np.random.default_rng(0).standard_normal(h.n)
x = sb.hbs_solve(h, b)
assert np.linalg.norm(sb.hbs_apply(h, x) - b) < 1e-9 * np.linalg.norm(b)
print("ok")
"""
    env = dict(os.environ, SBX_TEST_FAULT="far_prepare",
               PYTHONPATH=str(ROOT) + os.pathsep + os.environ.get("PYTHONPATH", ""))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr
