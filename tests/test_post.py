"""Boundary-patch post-processing (host, no GPU): flow_rate / patch_area / fit_loglog_slope against
values the reference produced on the same meshes and seeded fields (tests/golden/post.npz,
metrics.py:42-110)."""

import numpy as np
import pytest

from golden_util import golden
from paper_2009_06725_b200 import fit_loglog_slope, flow_rate, patch_area
from paper_2009_06725_b200.errors import MeshError
from paper_2009_06725_b200.workloads import c1_case, pipe3d_case


@pytest.fixture(scope="module")
def post():
    return golden("post.npz")


def _mesh(name):
    return c1_case().qmesh if name == "c1" else pipe3d_case().qmesh


@pytest.mark.parametrize("name", ["c1", "pipe3d"])
def test_flow_rate_and_area_match_reference(post, name):
    q = _mesh(name)
    assert np.array_equal(q.vel_conn, post[f"{name}_vel_conn"])   # same mesh as the reference's
    vec = post[f"{name}_vec"]
    patches = [k[len(f"{name}_area_"):] for k in post.files if k.startswith(f"{name}_area_")]
    assert patches
    for pn in patches:
        assert flow_rate(vec, q, pn) == pytest.approx(complex(post[f"{name}_flow_{pn}"]), rel=1e-12, abs=1e-14)
        fr = flow_rate(vec.real, q, pn)
        assert isinstance(fr, float)
        assert fr == pytest.approx(float(post[f"{name}_flowreal_{pn}"]), rel=1e-12, abs=1e-14)
        assert patch_area(q, pn) == pytest.approx(float(post[f"{name}_area_{pn}"]), rel=1e-13)


def test_unknown_patch_raises():
    with pytest.raises(MeshError):
        flow_rate(np.zeros((c1_case().qmesh.n_velocity_nodes, 2)), c1_case().qmesh, "nope")


def test_fit_loglog_slope(post):
    assert fit_loglog_slope(post["fit_x"], post["fit_y"]) == pytest.approx(float(post["fit_slope"]), rel=1e-13)
    with pytest.raises(ValueError):
        fit_loglog_slope([1.0, -1.0], [1.0, 2.0])
