"""Field snapshots (reference `io.py:88-183`): the native text format and
legacy-VTK output, written and read by the library's host runtime (`csrc/snapshot.cpp`).

Every float is printed with 17 significant digits exactly as the reference's ``"{:.17g}"``, so files
are byte-identical to the reference's and native snapshots round-trip bit-exactly; formatting and
parsing run in parallel on the host cores (10^7-10^8 values at configs 3-5).
"""

from __future__ import annotations

import os
from pathlib import Path

import numpy as np

from . import _lib
from .errors import ConfigError

__all__ = ["write_field_snapshot", "read_field_snapshot", "write_vtk_snapshot"]


def _c(path) -> bytes:
    return os.fsencode(str(Path(path)))


def _f64(a, shape=None):
    a = np.ascontiguousarray(a, dtype=float)
    if shape is not None:
        a = a.reshape(shape)
    return a


def write_field_snapshot(path, qmesh, velocity, pressure, fmt: str = "native", time: float | None = None) -> None:
    """Write a real nodal field in the native text format or legacy VTK (io.py:88-101)."""
    velocity = np.asarray(velocity, dtype=float)
    pressure = np.asarray(pressure, dtype=float)
    if velocity.shape != (qmesh.n_velocity_nodes, qmesh.dim):
        raise ValueError(f"velocity shape {velocity.shape} does not match the mesh")
    if pressure.shape != (qmesh.n_vertices,):
        raise ValueError(f"pressure shape {pressure.shape} does not match the mesh")
    if fmt == "native":
        t = 0.0 if time is None else float(time)
        nodes, v, p = _f64(qmesh.nodes), _f64(velocity), _f64(pressure)
        _lib.call("ss_write_snapshot", _c(path), qmesh.dim, qmesh.n_velocity_nodes, qmesh.n_vertices,
                  _lib.ptr(nodes), _lib.ptr(v), _lib.ptr(p), t)
    elif fmt == "vtk":
        write_vtk_snapshot(path, qmesh, velocity, pressure)
    else:
        raise ValueError(f"unknown snapshot format '{fmt}'")


def read_field_snapshot(path):
    """Read a native snapshot; returns ``(coords, velocity, pressure, time)`` (io.py:117-134)."""
    path = Path(path)
    with open(path) as fh:
        head = fh.readline().split()
    if len(head) != 5 or head[0] != "snapshot":
        raise ConfigError(f"{path}: not a native snapshot file")
    dim, n_v, n_p = int(head[1]), int(head[2]), int(head[3])
    time = float(head[4])
    coords = np.empty((n_v, dim))
    velocity = np.empty((n_v, dim))
    pressure = np.empty(n_p)
    try:
        _lib.call("ss_read_snapshot", _c(path), dim, n_v, n_p, _lib.ptr(coords), _lib.ptr(velocity),
                  _lib.ptr(pressure))
    except ValueError as exc:   # layout errors name the missing block, as the reference does
        raise ConfigError(f"{path}: {exc}") from None
    return coords, velocity, pressure, time


def write_vtk_snapshot(path, qmesh, velocity=None, pressure=None, title: str = "spectralstokes field") -> None:
    """Legacy-VTK ASCII unstructured grid with quadratic cells (io.py:140-183).  Pressure lives on
    vertices; mid-edge values are the averages of the edge endpoints."""
    nodes = _f64(qmesh.nodes)
    conn = np.ascontiguousarray(qmesh.vel_conn, dtype=np.int64)
    edges = np.ascontiguousarray(qmesh.edges, dtype=np.int64)
    v = None if velocity is None else _f64(velocity)
    p = None if pressure is None else _f64(pressure)
    _lib.call("ss_write_vtk", _c(path), title.encode(), qmesh.dim, qmesh.n_velocity_nodes, qmesh.n_vertices,
              _lib.ptr(nodes), len(conn), conn.shape[1], _lib.ptr(conn, _lib.C.c_int64),
              _lib.ptr(edges, _lib.C.c_int64), None if v is None else _lib.ptr(v), None if p is None else _lib.ptr(p))
