"""Install the B200 hot path under the reference's own import name, ``spectralstokes``.

The reference has no FFI or plugin registry; its boundary is the Python API re-exported by
``pkg/src/spectralstokes/__init__.py:10-46``.  :func:`install` makes that API run
on the device in one of two ways:

* **overlay** (the reference package is importable): its hot-path entry points are replaced in
  place -- ``assembly.assemble_mode_system`` (403-494), ``krylov.jacobi_precondition`` /
  ``gmres`` / ``gmres_solve`` (49-216), ``spectral._solve_one_mode`` / ``solve_modes`` /
  ``reconstruct`` / ``mode_energies`` / ``adaptive_mode_refinement`` (254-371) -- including the
  names other reference modules bound at import (``spectral``, ``runner``, the package root).
  Everything else (config, IO, CLI, the real-valued MSS path in ``timedomain``, which bound
  ``gmres`` before the overlay) keeps running the reference.  This package's exceptions and
  result types become the reference's own classes, so ``except spectralstokes.errors.MeshError``
  and ``isinstance(sol, spectralstokes.ModeSolution)`` hold for values produced on the GPU.
  The non-default ``viscous_form="symmetric"`` (assembly.py:206-229) is outside the B200 hot path
  (SURVEY.md §8a row 5); calls with it are passed to the reference's original function.
* **alias** (no reference installed, e.g. on a GPU box): ``spectralstokes`` and its submodules
  ``assembly``, ``krylov``, ``spectral``, ``mesh``, ``errors``, ``metrics``, ``structured``,
  ``io`` resolve to this package's modules.

:func:`uninstall` restores the previous state (tests use it).
"""

from __future__ import annotations

import importlib
import importlib.util
import sys

from . import _lib, assembly, boundary, errors, io, krylov, mesh, metrics, spectral, structured, vessels

NAME = "spectralstokes"
_OURS = [sys.modules[__package__], _lib, assembly, boundary, errors, io, krylov, mesh, metrics, spectral, structured, vessels]
_SUBMODULES = {"assembly": assembly, "krylov": krylov, "spectral": spectral, "mesh": mesh, "errors": errors,
               "metrics": metrics, "structured": structured, "io": io}

# reference module -> names replaced by this package's function of the same name
_OVERLAY = {
    "assembly": ["assemble_mode_system"],
    "krylov": ["jacobi_precondition", "gmres", "gmres_solve"],
    "spectral": ["assemble_mode_system", "gmres_solve", "solve_modes", "reconstruct", "mode_energies",
                 "adaptive_mode_refinement", "_solve_one_mode"],
    "runner": ["solve_modes", "reconstruct", "adaptive_mode_refinement"],
    "": ["assemble_mode_system", "jacobi_precondition", "gmres_solve", "solve_modes", "reconstruct",
         "adaptive_mode_refinement"],
}
# names in this package rebound to the reference's classes while the overlay is active
_SHARED_TYPES = {"MeshError": "errors", "ConfigError": "errors", "ConvergenceError": "errors",
                 "SolveReport": "krylov", "ModeSolution": "spectral"}

_state: dict | None = None


def _solve_one_mode(qmesh, props, mode_set, settings, idx, viscous_form):
    """``spectral._solve_one_mode`` (spectral.py:254-284) on the device: a one-mode batch."""
    from .spectral import ModeSet

    sub = ModeSet(indices=[int(idx)], frequencies=mode_set.frequencies, period=mode_set.period,
                  coefficients=mode_set.coefficients, waveforms=mode_set.waveforms)
    return spectral.solve_modes(qmesh, props, sub, settings, viscous_form=viscous_form)[0]


def _ours(name):
    table = {"assemble_mode_system": assembly.assemble_mode_system,
             "jacobi_precondition": krylov.jacobi_precondition, "gmres": krylov.gmres,
             "gmres_solve": krylov.gmres_solve, "solve_modes": spectral.solve_modes,
             "reconstruct": spectral.reconstruct, "mode_energies": spectral.mode_energies,
             "adaptive_mode_refinement": spectral.adaptive_mode_refinement, "_solve_one_mode": _solve_one_mode}
    return table[name]


def _with_form_passthrough(fn, original):
    """Device function for the full viscous form; the reference's original for any other form
    (``viscous_form`` given by keyword or position, per the reference's own signature)."""
    import inspect

    try:
        sig = inspect.signature(original if original is not None else fn)
    except (TypeError, ValueError):
        sig = None

    def wrapper(*args, **kwargs):
        form = kwargs.get("viscous_form", "full")
        if sig is not None and "viscous_form" not in kwargs:
            try:
                form = sig.bind_partial(*args, **kwargs).arguments.get("viscous_form", "full")
            except TypeError:
                pass
        if form != "full" and original is not None:
            return original(*args, **kwargs)
        return fn(*args, **kwargs)

    wrapper.__wrapped__ = fn
    wrapper.__name__ = getattr(fn, "__name__", "wrapper")
    wrapper.__doc__ = fn.__doc__
    return wrapper


def reference_available() -> bool:
    mod = sys.modules.get(NAME)
    if mod is not None:
        return not getattr(mod, "__b200_alias__", False)
    return importlib.util.find_spec(NAME) is not None


def install(mode: str = "auto"):
    """Make ``import spectralstokes`` run the hot path on the B200 library.

    ``mode``: "auto" (overlay when the reference is importable, else alias), "overlay", "alias".
    Returns the ``spectralstokes`` module.  Idempotent.
    """
    global _state
    if _state is not None:
        return sys.modules[NAME]
    if mode == "auto":
        mode = "overlay" if reference_available() else "alias"
    if mode == "alias":
        saved = {k: sys.modules.get(k) for k in [NAME] + [f"{NAME}.{s}" for s in _SUBMODULES]}
        pkg = sys.modules[__package__]
        pkg.__b200_alias__ = True
        sys.modules[NAME] = pkg
        for sub, mod in _SUBMODULES.items():
            sys.modules[f"{NAME}.{sub}"] = mod
        _state = {"mode": "alias", "saved_modules": saved}
        return pkg
    if mode != "overlay":
        raise ValueError(f"unknown install mode '{mode}'")
    ref = importlib.import_module(NAME)
    if getattr(ref, "__b200_alias__", False):
        raise RuntimeError("spectralstokes is already this package's alias")
    patched = []   # (module, name, previous value)
    for sub, names in _OVERLAY.items():
        rmod = ref if not sub else importlib.import_module(f"{NAME}.{sub}")
        for name in names:
            if not hasattr(rmod, name):
                continue
            prev = getattr(rmod, name)
            new = _ours(name)
            if name in ("assemble_mode_system", "solve_modes", "_solve_one_mode", "adaptive_mode_refinement"):
                new = _with_form_passthrough(new, prev)
            patched.append((rmod, name, prev))
            setattr(rmod, name, new)
    rebound = []
    for name, sub in _SHARED_TYPES.items():
        target = getattr(importlib.import_module(f"{NAME}.{sub}"), name)
        for mod in _OURS:
            if hasattr(mod, name):
                rebound.append((mod, name, getattr(mod, name)))
                setattr(mod, name, target)
    ref.__b200_overlay__ = True
    _state = {"mode": "overlay", "patched": patched, "rebound": rebound, "ref": ref}
    return ref


def uninstall():
    """Undo :func:`install`."""
    global _state
    if _state is None:
        return
    if _state["mode"] == "alias":
        for k, v in _state["saved_modules"].items():
            if v is None:
                sys.modules.pop(k, None)
            else:
                sys.modules[k] = v
        sys.modules[__package__].__b200_alias__ = False
    else:
        for mod, name, prev in reversed(_state["patched"]):
            setattr(mod, name, prev)
        for mod, name, prev in reversed(_state["rebound"]):
            setattr(mod, name, prev)
        _state["ref"].__b200_overlay__ = False
    _state = None


def installed_mode():
    return None if _state is None else _state["mode"]
