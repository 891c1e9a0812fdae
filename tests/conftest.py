"""Shared fixtures.  BLAS is pinned to one thread before numpy loads so the oracle reproduces the
reference's numbers run to run (the reference's own pkg/tests/conftest.py:5-9 does the same)."""

import os
import sys

os.environ.setdefault("OMP_NUM_THREADS", "1")
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("MKL_NUM_THREADS", "1")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import pytest  # noqa: E402

from paper_2009_06725_b200.mesh import BoundaryPatch, Mesh, promote_to_quadratic  # noqa: E402
from paper_2009_06725_b200.structured import channel_grid  # noqa: E402

def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests through the C ABI")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture
def fluid():
    from paper_2009_06725_b200.assembly import FluidProps

    return FluidProps(density=1.0, viscosity=1.0)


@pytest.fixture
def small_channel_qmesh():
    """channel_grid(10, 4) on [0,4]x[-1,1] (reference conftest.py:62-65)."""
    return promote_to_quadratic(channel_grid(10, 4, length=4.0, half_height=1.0))


@pytest.fixture
def single_triangle_qmesh():
    nodes = np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0]])
    patches = {"boundary": BoundaryPatch(kind="wall", faces=np.array([[0, 1], [1, 2], [2, 0]]))}
    return promote_to_quadratic(Mesh(nodes, np.array([[0, 1, 2]]), patches))
