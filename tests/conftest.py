import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libhjb200.so")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def pytest_collection_modifyitems(config, items):
    try:
        import torch

        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(params=["auto", "brick_always", "generic", "tile_stages", "axes"])
def stage_kernel(request):
    """Run a GPU parity test under every fused-stage kernel family: the
    default dispatch (small grids: the tile kernel, an integration interval
    in one persistent launch; large WENO5 grids: the per-axis walk
    pipeline), the brick kernels forced even on tiny grids, the per-node
    generic kernel, the tile kernel launched per stage, and the per-axis
    walk pipeline forced on every size."""
    from paper_2411_03501_b200 import device as dev

    old = dev.set_stage_kernel(request.param)
    yield request.param
    dev.set_stage_kernel(old)
