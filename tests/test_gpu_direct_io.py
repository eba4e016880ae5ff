"""One-right-hand-side sweeps read and write the caller's device vectors
directly (no copy into the sweep workspace, sweep.cu SweepDirectIo) and the
dataflow kernel zeroes its own dependency counters.  hbs.cpp:511-664
(hbs_apply / hbs_solve and their transposes) are the functions behind it."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def setup():
    import torch
    import paper_2108_07205_b200 as sb
    sb.init(0)
    g = sb.panelize(sb.star(5, 0.3), 96, 16)
    h = sb.hbs_invert(sb.hbs_compress(g, opts=sb.HbsOptions(eps=1e-10)))
    return sb, torch, h


def test_one_rhs_equals_a_column_of_a_block(setup):
    """The direct 1-RHS GEMV sweep against the DMMA sweep of a 3-column block
    (workspace path) and the host-pointer path, repeated calls included (the
    counters the kernel resets itself must be clean for every launch)."""
    sb, torch, h = setup
    n = h.info()["n"]
    rng = np.random.default_rng(5)
    B = rng.uniform(-1, 1, (n, 3))
    X3 = sb.hbs_solve(h, B)
    stream = torch.cuda.ExternalStream(sb.api.lib().sbx_stream())
    for rep in range(4):
        for transpose in (False, True):
            ref = sb.hbs_solve(h, B[:, 1].copy(), transpose=transpose)  # host pointers
            with torch.cuda.stream(stream):
                x = sb.hbs_solve(h, torch.from_numpy(B[:, 1].copy()).cuda(), transpose=transpose)
                x = x.cpu().numpy()
            assert np.array_equal(x, ref)
            if not transpose:
                assert np.linalg.norm(x - X3[:, 1]) <= 1e-12 * np.linalg.norm(x)
        with torch.cuda.stream(stream):
            y = sb.hbs_apply(h, torch.from_numpy(X3[:, 1].copy()).cuda()).cpu().numpy()
        assert np.linalg.norm(y - B[:, 1]) <= 1e-8 * np.linalg.norm(B[:, 1])


def test_in_place_call_falls_back_to_the_workspace_path(setup):
    """x == b (overlapping vectors) must not take the direct path."""
    sb, torch, h = setup
    from paper_2108_07205_b200 import _sbx
    n = h.info()["n"]
    b = np.random.default_rng(6).uniform(-1, 1, n)
    ref = sb.hbs_solve(h, b)
    stream = torch.cuda.ExternalStream(sb.api.lib().sbx_stream())
    with torch.cuda.stream(stream):
        t = torch.from_numpy(b.copy()).cuda()
        for flags in (_sbx.SBX_DEVICE_PTRS, _sbx.SBX_DEVICE_PTRS | _sbx.SBX_ROW_MAJOR):
            t.copy_(torch.from_numpy(b))
            ld = 1 if flags & _sbx.SBX_ROW_MAJOR else n
            sb.api.check(sb.api.lib().sbx_hbs_solve(h.ptr, C.c_void_p(t.data_ptr()), ld, 1,
                                                    C.c_void_p(t.data_ptr()), ld, flags,
                                                    C.c_void_p(sb.api.lib().sbx_stream())))
            assert np.array_equal(t.cpu().numpy(), ref)
