"""The C-ABI library builds, loads and exports every symbol declared in include/*.h.

No GPU needed: only host-side entry points are called (reference tables, traction load).
"""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

import oracle
from paper_2009_06725_b200 import _lib
from paper_2009_06725_b200.assembly import boundary_traction_load, reference_shapes
from golden_util import golden

ROOT = Path(__file__).resolve().parent.parent


def _declared_symbols():
    names = set()
    for h in (ROOT / "include").glob("*.h"):
        text = re.sub(r"/\*.*?\*/", "", h.read_text(), flags=re.S)
        names |= set(re.findall(r"\b(ss_[a-z0-9_]+)\s*\(", text))
    return sorted(names)


def test_header_declares_the_entry_points():
    names = _declared_symbols()
    for required in ("ss_pattern_create", "ss_assemble", "ss_spmv_batched", "ss_krylov_solve", "ss_reconstruct",
                     "ss_rhs_batched", "ss_pattern_export", "ss_last_error"):
        assert required in names


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    missing = [n for n in _declared_symbols() if not hasattr(lib, n)]
    assert not missing, missing
    assert set(_lib.SIGNATURES) >= set(_declared_symbols())


def _declared_arity():
    """Parameter count of every ss_* function declared in include/*.h."""
    out = {}
    for h in (ROOT / "include").glob("*.h"):
        text = re.sub(r"/\*.*?\*/", "", h.read_text(), flags=re.S)
        for name, params in re.findall(r"\b(ss_[a-z0-9_]+)\s*\(([^)]*)\)\s*;", text):
            p = params.strip()
            out[name] = 0 if p in ("", "void") else p.count(",") + 1
    return out


def test_ctypes_signatures_match_header_arity():
    """The ctypes table and the C header agree on every entry point's parameter count."""
    arity = _declared_arity()
    assert len(arity) >= 40
    bad = {n: (len(_lib.SIGNATURES[n][1]), a) for n, a in arity.items()
           if n in _lib.SIGNATURES and len(_lib.SIGNATURES[n][1]) != a}
    assert not bad, bad


def test_library_is_sm100a_code():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("dim", [2, 3])
def test_native_reference_tables_match_reference(dim):
    g = golden("shapes.npz")
    nv, npr = (6, 3) if dim == 2 else (10, 4)
    m = np.zeros(nv * nv)
    s = np.zeros(nv * nv * dim * dim)
    t = np.zeros(nv * dim * npr)
    _lib.call("ss_reference_tables", dim, _lib.ptr(m), _lib.ptr(s), _lib.ptr(t))
    np.testing.assert_allclose(m.reshape(nv, nv), g[f"d{dim}_mref"], rtol=0, atol=2e-16)
    np.testing.assert_allclose(s.reshape(nv, nv, dim, dim), g[f"d{dim}_sref"], rtol=0, atol=2e-15)
    np.testing.assert_allclose(t.reshape(nv, dim, npr), g[f"d{dim}_tref"], rtol=0, atol=2e-16)


@pytest.mark.parametrize("dim", [2, 3])
def test_reference_shapes_api(dim):
    g = golden("shapes.npz")
    s = reference_shapes(dim)
    assert np.array_equal(s.points, g[f"d{dim}_points"]) and np.array_equal(s.weights, g[f"d{dim}_weights"])
    np.testing.assert_allclose(s.vel_grads, g[f"d{dim}_vel_grads"], atol=1e-15)
    with pytest.raises(ValueError):
        reference_shapes(4)
    with pytest.raises(ValueError):
        reference_shapes(2, quadrature_order=2)


def test_traction_load_matches_oracle(small_channel_qmesh):
    q = small_channel_qmesh
    for h in (np.array([1.0 + 0.5j, -0.25j]), np.arange(8).reshape(4, 2) * (1 + 1j),
              (q.nodes[:, :1] * np.array([[1.0, 2.0]])).astype(complex)):
        mine = boundary_traction_load(q, "inlet", h)
        ref = oracle.surface_load(q, "inlet", h)
        np.testing.assert_allclose(mine, ref, rtol=1e-14, atol=1e-15)
    load = boundary_traction_load(q, "inlet", np.array([1.0 + 0j, 0.0]))
    assert load[:, 0].sum() == pytest.approx(2.0, rel=1e-12)


def test_traction_load_3d_matches_oracle():
    from paper_2009_06725_b200.mesh import promote_to_quadratic
    from paper_2009_06725_b200.structured import pipe_grid

    m, geom = pipe_grid(2, 2, 0.5, 1.0)
    q = promote_to_quadratic(m, geom)
    for h in (np.array([0.0, 0.3, 1.0 - 2j]), (q.nodes * np.array([1.0, 0.5, 2.0])).astype(complex)):
        np.testing.assert_allclose(boundary_traction_load(q, "outlet", h), oracle.surface_load(q, "outlet", h),
                                   rtol=1e-13, atol=1e-15)


def test_traction_errors(small_channel_qmesh):
    from paper_2009_06725_b200.errors import MeshError

    with pytest.raises(MeshError, match="neumann"):
        boundary_traction_load(small_channel_qmesh, "walls", np.array([1.0, 0.0]))
    with pytest.raises(MeshError):
        boundary_traction_load(small_channel_qmesh, "nope", np.array([1.0, 0.0]))
    with pytest.raises(ValueError):
        boundary_traction_load(small_channel_qmesh, "inlet", np.zeros(5))


def test_no_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2009_06725_b200.errors import DeviceError
    from paper_2009_06725_b200 import solve_modes, FluidProps
    from paper_2009_06725_b200.mesh import promote_to_quadratic
    from paper_2009_06725_b200.structured import channel_grid
    from paper_2009_06725_b200.spectral import BoundaryWaveform, fourier_transform_bcs

    q = promote_to_quadratic(channel_grid(4, 2))
    wf = BoundaryWaveform("inlet", "neumann", [1.0, 0.0], 1.0, coefficients=[1.0, 0.5])
    with pytest.raises(DeviceError):
        solve_modes(q, FluidProps(1.0, 1.0), fourier_transform_bcs([wf], 1))
