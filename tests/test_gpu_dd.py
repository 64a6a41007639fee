"""The NCCL data plane of the slab decomposition (hj_dd_*, csrc/hj_dd.cu) on
one GPU.  A single slab of a periodic axis 0 is a one-rank ring: its halo
planes travel through libhjb200's own NCCL communicator (grouped
ncclSend/ncclRecv to itself on the exchange stream, the CORE launch
meanwhile, then RIM) instead of the kernels' periodic wrap.  The result must
equal the undecomposed run bit for bit -- the same code path every rank runs
on 2/4/8 GPUs, with no kernel waiting on another rank's kernel."""
import ctypes

import numpy as np
import pytest

import paper_2411_03501_b200 as hj
from paper_2411_03501_b200 import _lib
from paper_2411_03501_b200 import device as dev
from paper_2411_03501_b200.distributed import NcclTransport, SlabIntegrator, partition
from paper_2411_03501_b200.engine import FusedIntegrator

pytestmark = pytest.mark.gpu


def _periodic3(n=(40, 20, 24)):
    g = hj.create_grid((0.0, -1.0, -1.0), (2 * np.pi, 1.0, 1.0), n, periodic_axes={0})
    x = g.axis_nodes[0][:, None, None]
    y0 = np.sin(x) + 0.1 * np.cos(3 * g.axis_nodes[1][None, :, None]) + 0.05 * g.axis_nodes[2][None, None, :]
    return g, y0


def _steps(run, y, dt, k):
    t = 0.0
    for _ in range(k):
        y = run.step3(y, t, dt)
        t += dt
    return y


@pytest.mark.parametrize("overlap", [True, False])
@pytest.mark.parametrize("scheme", ["weno5", "eno2"])
def test_self_ring_equals_single_domain(overlap, scheme):
    g, y0 = _periodic3()
    cfg = hj.advection_term_config([1.0, -0.5, 0.25], scheme=scheme)
    dt = 0.5 / float(np.sum(cfg.partials.alphas(0.0, g) / g.spacings))
    ref = dev.to_host(_steps(FusedIntegrator(g, cfg), dev.to_dev(y0), dt, 3))
    run = SlabIntegrator(g, cfg, 0, 1, transport="nccl", overlap=overlap, self_ring=True)
    assert isinstance(run.transport, NcclTransport)
    got = _steps(run, run.scatter(y0), dt, 3)
    assert np.array_equal(ref, dev.to_host(run.owned(got)))
    ex, by = run.transport.traffic()
    plane = int(np.prod(g.counts[1:]))
    assert ex == 9 and by == 9 * 2 * 3 * plane * 8     # 3 steps x 3 stages, 3 planes each way
    run.transport.close()


def test_self_ring_4d():
    g = hj.create_grid((0.0, -1.0, -1.0, -1.0), (2 * np.pi, 1.0, 1.0, 1.0), (24, 12, 17, 18), periodic_axes={0})
    cfg = hj.advection_term_config([0.5, -0.25, 0.75, 1.0], scheme="weno5")
    x = g.axis_nodes[0][:, None, None, None]
    y0 = np.cos(x) + 0.2 * g.axis_nodes[3][None, None, None, :] + 0.0 * g.axis_nodes[1][None, :, None, None]
    y0 = np.broadcast_to(y0, g.counts).copy()
    dt = 0.5 / float(np.sum(cfg.partials.alphas(0.0, g) / g.spacings))
    ref = dev.to_host(_steps(FusedIntegrator(g, cfg), dev.to_dev(y0), dt, 2))
    run = SlabIntegrator(g, cfg, 0, 1, transport="nccl", self_ring=True)
    got = _steps(run, run.scatter(y0), dt, 2)
    assert np.array_equal(ref, dev.to_host(run.owned(got)))


def test_self_ring_interval_with_mask_and_error_path():
    """integrate() over an interval (the tube's mask in the last stage) through
    hj_dd_stage, then a non-finite input: the all-reduced stats raise exactly
    the single-domain error."""
    g, y0 = _periodic3((32, 18, 20))
    cfg = hj.advection_term_config([1.0, 0.5, -0.25], scheme="weno5")
    opts = hj.IntegratorOptions()
    single = FusedIntegrator(g, cfg)
    ref = single.integrate(3, (0.0, 0.2), dev.to_dev(y0), opts, mask_prev=dev.to_dev(y0), use_min=True)
    run = SlabIntegrator(g, cfg, 0, 1, transport="nccl", self_ring=True)
    buf = run.scatter(y0)
    got = run.integrate(3, (0.0, 0.2), buf, opts, mask_prev=buf, use_min=True)
    assert got.steps_taken == ref.steps_taken and got.t_final == ref.t_final
    assert np.array_equal(dev.to_host(ref.y), dev.to_host(run.owned(got.y)))
    bad = y0.copy()
    bad[5, 3, 4] = np.nan
    with pytest.raises(Exception) as e1:
        single.integrate(3, (0.0, 0.2), dev.to_dev(bad), opts)
    with pytest.raises(Exception) as e2:
        run.integrate(3, (0.0, 0.2), run.scatter(bad), opts)
    assert type(e1.value) is type(e2.value) and str(e1.value) == str(e2.value)


def test_gather_and_reduce_on_one_rank():
    g, y0 = _periodic3((24, 10, 12))
    cfg = hj.advection_term_config([1.0, 0.5, -0.25], scheme="weno5")
    run = SlabIntegrator(g, cfg, 0, 1, transport="nccl", self_ring=True)
    buf = run.scatter(y0)
    full = run.transport.gather(partition(24, 1, 3, True, self_ring=True), run.owned(buf), 0)
    assert np.array_equal(full, y0)
    st = dev.Stats().reset()
    merged = run.transport.merge_stats(st)
    assert merged.nonfinite == 0 and merged.first_bad_tag == 0x7FFFFFFF
    assert _lib.load().hj_dd_nccl_version() > 0


def test_abi_rejects_thin_halo_and_missing_neighbour():
    lib = _lib.load()
    g, y0 = _periodic3((24, 10, 12))
    cfg = hj.advection_term_config([1.0, 0.5, -0.25], scheme="weno5")
    with pytest.raises(ValueError, match="halo"):
        SlabIntegrator(g, cfg, 0, 1, halo=2, transport="nccl", self_ring=True)
    # a communicator without neighbours cannot serve a grid that expects halos
    uid = ctypes.create_string_buffer(_lib.DD_UID_BYTES)
    _lib.check(lib.hj_dd_unique_id(uid), "uid")
    h = ctypes.c_void_p()
    _lib.check(lib.hj_dd_init(uid, 1, 0, -1, -1, ctypes.byref(h)), "init")
    try:
        dg = dev.DeviceGrid(g, slab=(0, 24, 1, 1, 3))
        v = dev.to_dev(np.zeros((30, 10, 12)))
        rc = lib.hj_dd_exchange(h, dg.ref, dev.ptr(v[3:]), dev.stream())
        assert rc == _lib.HJ_EINVAL and b"neighbour" in lib.hj_last_error()
    finally:
        lib.hj_dd_free(h)


@pytest.mark.parametrize("dim", [3, 4])
def test_self_ring_per_axis_pipeline(dim):
    """The slab stage on the per-axis walk pipeline (hj_dd_stage: the
    contiguous-axis kernel overlaps the exchange, the column kernels follow
    it), forced on a small grid, against the single domain under the same
    kernel family and under the default dispatch."""
    if dim == 3:
        g, y0 = _periodic3()
        cfg = hj.advection_term_config([1.0, -0.5, 0.25], scheme="weno5")
    else:
        g = hj.create_grid((0.0, -1.0, -1.0, -1.0), (2 * np.pi, 1.0, 1.0, 1.0), (24, 12, 17, 18),
                           periodic_axes={0})
        cfg = hj.advection_term_config([0.5, -0.25, 0.75, 1.0], scheme="weno5")
        x = g.axis_nodes[0][:, None, None, None]
        y0 = np.broadcast_to(np.cos(x) + 0.2 * g.axis_nodes[3][None, None, None, :], g.counts).copy()
    dt = 0.5 / float(np.sum(cfg.partials.alphas(0.0, g) / g.spacings))
    old = dev.set_stage_kernel("axes")
    try:
        ref = dev.to_host(_steps(FusedIntegrator(g, cfg), dev.to_dev(y0), dt, 2))
        run = SlabIntegrator(g, cfg, 0, 1, transport="nccl", overlap=True, self_ring=True)
        got = dev.to_host(run.owned(_steps(run, run.scatter(y0), dt, 2)))
        run.transport.close()
    finally:
        dev.set_stage_kernel(old)
    default = dev.to_host(_steps(FusedIntegrator(g, cfg), dev.to_dev(y0), dt, 2))
    assert np.array_equal(ref, got)
    assert np.array_equal(default, got)
