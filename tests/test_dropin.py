"""The drop-in under the reference's own import name (paper_2009_06725_b200.dropin).

* overlay (CPU, needs /root/reference -- present in the build container only): the reference
  package's hot-path names are replaced by this package's functions, and the exceptions this
  package raises are the reference's own classes (``except spectralstokes.errors.MeshError``);
  ``uninstall`` restores the reference.
* alias (GPU): with no reference installed, ``import spectralstokes`` gives this package and its
  solve path runs on the device.
"""

import importlib
import os
import sys

import numpy as np
import pytest

REF_SRC = "/root/reference/pkg/src"


@pytest.fixture
def reference_on_path():
    if not os.path.isdir(os.path.join(REF_SRC, "spectralstokes")):
        pytest.skip("reference package not present (only in the build container)")
    old_path = list(sys.path)
    saved = {k: v for k, v in sys.modules.items() if k == "spectralstokes" or k.startswith("spectralstokes.")}
    sys.path.insert(0, REF_SRC)
    for k in saved:
        del sys.modules[k]
    sys.dont_write_bytecode = True
    yield
    from paper_2009_06725_b200 import dropin

    dropin.uninstall()
    for k in [k for k in sys.modules if k == "spectralstokes" or k.startswith("spectralstokes.")]:
        del sys.modules[k]
    sys.modules.update(saved)
    sys.path[:] = old_path


def test_overlay_replaces_hot_path_and_shares_exception_types(reference_on_path):
    import paper_2009_06725_b200 as b2
    from paper_2009_06725_b200 import dropin

    ref = dropin.install()
    assert dropin.installed_mode() == "overlay"
    import spectralstokes

    assert spectralstokes is ref and not getattr(spectralstokes, "__b200_alias__", False)
    assert spectralstokes.krylov.gmres_solve is b2.krylov.gmres_solve
    assert spectralstokes.krylov.jacobi_precondition is b2.krylov.jacobi_precondition
    assert spectralstokes.spectral.reconstruct is b2.spectral.reconstruct
    for name in ("solve_modes", "assemble_mode_system", "adaptive_mode_refinement"):
        assert getattr(spectralstokes, name).__wrapped__ is getattr(b2, name)
    assert spectralstokes.runner.solve_modes.__wrapped__ is b2.spectral.solve_modes
    # the out-of-scope "symmetric" viscous form goes to the reference's own function, whether
    # passed by keyword or by position
    calls = []
    wrapped = spectralstokes.spectral._solve_one_mode
    orig = dropin._state["patched"]
    prev = next(p for m, n, p in orig if m is spectralstokes.spectral and n == "_solve_one_mode")
    import functools

    spy = functools.wraps(prev)(lambda *a, **k: calls.append((a, k)) or "ref")
    w2 = dropin._with_form_passthrough(wrapped.__wrapped__, spy)
    assert w2(None, None, None, None, 1, "symmetric") == "ref"
    assert w2(None, None, None, None, 1, viscous_form="symmetric") == "ref" and len(calls) == 2
    # the MSS time-domain path bound gmres at import and stays on the reference's CPU code
    assert spectralstokes.timedomain.gmres is not b2.krylov.gmres
    # exceptions raised by this package are the reference's classes
    from paper_2009_06725_b200.mesh import promote_to_quadratic
    from paper_2009_06725_b200.structured import channel_grid

    q = promote_to_quadratic(channel_grid(4, 2, length=2.0, half_height=1.0))
    with pytest.raises(spectralstokes.errors.MeshError):
        b2.boundary_traction_load(q, "no_such_patch", np.array([1.0, 0.0]))
    with pytest.raises(spectralstokes.MeshError):
        b2.boundary_traction_load(q, "walls" if "walls" in q.boundary_patches else "wall", np.array([1.0, 0.0]))
    # the reference's own mesh objects feed the drop-in host path unchanged
    rs = importlib.import_module("spectralstokes.structured")
    rq = spectralstokes.promote_to_quadratic(rs.channel_grid(4, 2, length=2.0, half_height=1.0))
    load_ref = importlib.import_module("spectralstokes.assembly")
    assert np.allclose(b2.boundary_traction_load(rq, "inlet", np.array([1.0, 0.0])),
                       load_ref.boundary_traction_load(rq, "inlet", np.array([1.0, 0.0])), rtol=1e-14, atol=1e-15)
    dropin.uninstall()
    assert dropin.installed_mode() is None
    assert spectralstokes.krylov.gmres_solve is not b2.krylov.gmres_solve
    assert b2.errors.MeshError is not spectralstokes.errors.MeshError
    assert b2.mesh.MeshError is b2.errors.MeshError


def test_alias_when_reference_absent():
    from paper_2009_06725_b200 import dropin

    if dropin.reference_available():
        pytest.skip("a reference spectralstokes is importable here (overlay mode applies)")
    mod = dropin.install()
    try:
        import spectralstokes
        import spectralstokes.krylov as sk

        assert spectralstokes is mod and sk.gmres_solve is mod.krylov.gmres_solve
        assert spectralstokes.MeshError is mod.errors.MeshError
    finally:
        dropin.uninstall()
    assert "spectralstokes" not in sys.modules


@pytest.mark.gpu
def test_alias_solves_on_the_device():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2009_06725_b200 import dropin

    if dropin.reference_available():
        pytest.skip("a reference spectralstokes is importable here (overlay mode applies)")
    dropin.install()
    try:
        import spectralstokes as ss
        from paper_2009_06725_b200 import _lib

        q = ss.mesh.promote_to_quadratic(ss.structured.channel_grid(10, 4, length=4.0, half_height=1.0))
        wf = ss.BoundaryWaveform("inlet", "neumann", np.array([1.0, 0.0]), 1.0, coefficients=np.array([0.3, 1.0]))
        l0 = _lib.launch_count()
        sols = ss.solve_modes(q, ss.FluidProps(1.0, 1.0), ss.fourier_transform_bcs([wf], 1),
                              ss.SolverSettings(tolerance=1e-10))
        assert _lib.launch_count() > l0
        assert all(s.report.converged for s in sols)
        with pytest.raises(ss.errors.MeshError):
            ss.assembly.boundary_traction_load(q, "nope", np.array([1.0, 0.0]))
    finally:
        dropin.uninstall()
