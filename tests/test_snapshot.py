"""Field snapshots (host runtime, no GPU): byte-identical to files the reference wrote for the same
meshes and fields (tests/golden/snap.npz, io.py:88-183), and bit-exact native round trips
(the reference's test_io_cli.py:97-112 contract)."""

import numpy as np
import pytest

from golden_util import golden
from paper_2009_06725_b200.errors import ConfigError
from paper_2009_06725_b200.io import read_field_snapshot, write_field_snapshot, write_vtk_snapshot
from paper_2009_06725_b200.mesh import promote_to_quadratic
from paper_2009_06725_b200.structured import channel_grid, pipe_grid


@pytest.fixture(scope="module")
def snap():
    return golden("snap.npz")


def _mesh(name):
    if name == "chan":
        return promote_to_quadratic(channel_grid(3, 2, 2.0, 1.0))
    m, geom = pipe_grid(2, 3, 0.5, 5.0)
    return promote_to_quadratic(m, geom)


@pytest.mark.parametrize("name", ["chan", "pipe"])
def test_snapshot_bytes_match_reference(tmp_path, snap, name):
    q = _mesh(name)
    assert np.array_equal(q.vel_conn, snap[f"{name}_vel_conn"])
    vel, pres = snap[f"{name}_vel"], snap[f"{name}_pres"]
    for fmt in ("native", "vtk"):
        path = tmp_path / f"{name}.{fmt}"
        write_field_snapshot(path, q, vel, pres, fmt=fmt, time=0.375)
        assert path.read_bytes() == snap[f"{name}_{fmt}_bytes"].tobytes(), fmt
    path = tmp_path / f"{name}_geom.vtk"
    write_vtk_snapshot(path, q, title="geometry only")
    assert path.read_bytes() == snap[f"{name}_vtkgeom_bytes"].tobytes()


@pytest.mark.parametrize("name", ["chan", "pipe"])
def test_native_roundtrip_bit_identical(tmp_path, snap, name):
    q = _mesh(name)
    vel, pres = snap[f"{name}_vel"], snap[f"{name}_pres"]
    path = tmp_path / "snap.txt"
    write_field_snapshot(path, q, vel, pres, time=0.125)
    coords, v2, p2, t = read_field_snapshot(path)
    assert np.array_equal(v2, vel) and np.array_equal(p2, pres) and t == 0.125
    assert np.array_equal(np.signbit(p2), np.signbit(pres))
    assert np.array_equal(coords, q.nodes)
    path2 = tmp_path / "snap2.txt"
    write_field_snapshot(path2, q, v2, p2, time=t)
    assert path.read_bytes() == path2.read_bytes()


def test_snapshot_errors(tmp_path):
    q = _mesh("chan")
    with pytest.raises(ValueError, match="velocity shape"):
        write_field_snapshot(tmp_path / "a", q, np.zeros((3, 2)), np.zeros(q.n_vertices))
    with pytest.raises(ValueError, match="pressure shape"):
        write_field_snapshot(tmp_path / "a", q, np.zeros((q.n_velocity_nodes, 2)), np.zeros(2))
    with pytest.raises(ValueError, match="unknown snapshot format"):
        write_field_snapshot(tmp_path / "a", q, np.zeros((q.n_velocity_nodes, 2)), np.zeros(q.n_vertices), fmt="x")
    bad = tmp_path / "bad.txt"
    bad.write_text("hello\n")
    with pytest.raises(ConfigError, match="not a native snapshot"):
        read_field_snapshot(bad)
    write_field_snapshot(tmp_path / "ok.txt", q, np.zeros((q.n_velocity_nodes, 2)), np.zeros(q.n_vertices))
    text = (tmp_path / "ok.txt").read_text().replace("pressure\n", "presure\n")
    (tmp_path / "broken.txt").write_text(text)
    with pytest.raises(ConfigError, match="missing pressure block"):
        read_field_snapshot(tmp_path / "broken.txt")
