"""Drop-in Krylov API on the device GMRES engine (reference `krylov.py`).

``SolverSettings`` (19-34), ``SolveReport`` (37-46), ``jacobi_precondition`` (49-60), ``gmres``
(63-164) and ``gmres_solve`` (171-216) keep their names, signatures, defaults and error
behaviour.  The iteration itself runs in `csrc/krylov.cu`: a mode-batched, graph-captured,
device-resident restarted GMRES with the reference's CGS2 + Givens + true-residual semantics.
``gmres_batched`` is the batched entry point used by ``solve_modes``.
"""

from __future__ import annotations

import ctypes as C
import os
import time
import weakref
from dataclasses import dataclass, field

import numpy as np

from . import _lib

__all__ = ["SolverSettings", "SolveReport", "jacobi_precondition", "gmres", "gmres_solve", "gmres_batched",
           "KrylovWorkspace", "MAX_RESTART"]

# Largest restart served by the shared-memory-ring basis passes; larger restarts (any value >= 1, as
# the reference accepts, krylov.py:24,31-32) run the wide passes that read the basis from global memory.
MAX_RESTART = 240


@dataclass
class SolverSettings:
    """Iterative solve controls (krylov.py:19-34)."""

    tolerance: float = 1e-6
    restart: int = 200
    max_iterations: int = 200_000
    preconditioner: str = "jacobi"

    def __post_init__(self):
        if not 0.0 < self.tolerance < 1.0:
            raise ValueError("tolerance must lie in (0, 1)")
        if self.restart < 1:
            raise ValueError("restart must be at least 1")
        if self.preconditioner not in ("none", "jacobi"):
            raise ValueError(f"unknown preconditioner '{self.preconditioner}'")


@dataclass
class SolveReport:
    """Outcome of one linear solve (krylov.py:37-46).

    For batched solves ``wall_time``/``cpu_time`` are the batch call's, scaled by the fraction of the
    batch's ticks the mode needed (modes finish at their own tick).
    """

    iterations: int
    residual: float
    converged: bool
    wall_time: float
    cpu_time: float = 0.0
    residual_history: list = field(default_factory=list, repr=False)


class KrylovWorkspace:
    """Owns one ``ss_krylov`` handle (basis Q, Hessenberg, per-mode state, cached graphs)."""

    def __init__(self, handle, device, restart, max_batch, hist_cap, n, keep=None):
        self._h = handle
        self.device = device
        self.restart = restart
        self.max_batch = max_batch
        self.hist_cap = hist_cap
        self.n = n
        self._keep = keep
        info = np.zeros(10, dtype=np.int64)
        _lib.call("ss_krylov_info", handle, _lib.ptr(info, C.c_int64))
        self.info = info
        self.ld = int(info[1])
        self._finalizer = weakref.finalize(self, _lib.load().ss_krylov_destroy, handle)

    def close(self):
        self._finalizer()

    def set_option(self, name: str, value: int):
        """Native workspace option (``ss_krylov_set_option``): "row_spmv", "device_loop", "ticks_per_graph", "fused", "pass_alt"."""
        _lib.call("ss_krylov_set_option", self._h, name.encode(), int(value))

    def options(self):
        out = {}
        for name in ("row_spmv", "stream_spmv", "device_loop", "ticks_per_graph", "fused", "fused_active", "pass_alt"):
            v = C.c_int64()
            _lib.call("ss_krylov_get_option", self._h, name.encode(), C.byref(v))
            out[name] = int(v.value)
        return out

    @classmethod
    def for_operator(cls, op, restart: int, max_batch: int, hist_cap: int):
        h = C.c_void_p()
        _lib.call("ss_krylov_create_saddle", op.handle, int(max_batch), int(restart), int(hist_cap), C.byref(h))
        return cls(h, op.device, restart, max_batch, hist_cap, op.n, keep=op)

    @classmethod
    def for_csr(cls, matrix, restart: int, max_batch: int, hist_cap: int, scale=None, jacobi_from_diag=False,
                device=None):
        import scipy.sparse as sp

        torch = _lib.torch_mod()
        dev = torch.cuda.current_device() if device is None else int(device)
        a = sp.csr_matrix(matrix, dtype=complex)
        n = a.shape[0]
        ip = np.ascontiguousarray(a.indptr, dtype=np.int32)
        ix = np.ascontiguousarray(a.indices, dtype=np.int32)
        vals = np.ascontiguousarray(a.data, dtype=complex)
        sc = None if scale is None else np.ascontiguousarray(np.asarray(scale, dtype=complex).ravel())
        h = C.c_void_p()
        _lib.call("ss_krylov_create_csr", dev, n, int(a.nnz), _lib.ptr(ip, C.c_int32), _lib.ptr(ix, C.c_int32), 1,
                  _lib.ptr(vals.view(np.float64)), None if sc is None else _lib.ptr(sc.view(np.float64)),
                  int(bool(jacobi_from_diag)), int(max_batch), int(restart), int(hist_cap), C.byref(h))
        return cls(h, torch.device("cuda", dev), restart, max_batch, hist_cap, n)

    def csr_scale(self):
        out = np.zeros(self.n, dtype=complex)
        _lib.call("ss_krylov_csr_scale", self._h, 0, _lib.ptr(out.view(np.float64)))
        return out

    def solve(self, omegas, rhs, x0=None, tol=1e-6, maxiter=200_000, jacobi=True, x_out=None):
        """Solve ``len(omegas)`` modes; rhs/x0/x_out are (nb, ld) complex128 device tensors."""
        torch = _lib.torch_mod()
        om = np.ascontiguousarray(np.asarray(omegas, dtype=float).reshape(-1))
        nb = om.size
        if nb > self.max_batch:
            raise ValueError("batch larger than the workspace")
        x = x_out if x_out is not None else torch.zeros((nb, self.ld), dtype=torch.complex128, device=self.device)
        if x0 is not None and x0.data_ptr() != x.data_ptr():
            x.copy_(x0)
        oi = np.zeros(6 * nb, dtype=np.int64)
        od = np.zeros(4 * nb, dtype=np.float64)
        _lib.call("ss_krylov_solve", self._h, nb, _lib.ptr(om), None, _lib.dptr(rhs), _lib.dptr(x), self.ld,
                  int(x0 is not None), float(tol), int(maxiter), int(bool(jacobi)), _lib.stream_ptr(self.device),
                  _lib.ptr(oi, C.c_int64), _lib.ptr(od))
        oi = oi.reshape(nb, 6)
        od = od.reshape(nb, 4)
        return dict(x=x, iterations=oi[:, 0].copy(), converged=oi[:, 1].astype(bool), breakdown=oi[:, 2].astype(bool),
                    hist_len=oi[:, 4].copy(), zero_rhs=oi[:, 5].astype(bool), cycle_residual=od[:, 0].copy(),
                    estimate=od[:, 1].copy(), bnorm=od[:, 2].copy(), target=od[:, 3].copy())

    def residuals(self, nb: int) -> np.ndarray:
        """True relative residuals of the workspace's current X (device, fixed-order sums)."""
        out = np.zeros(nb)
        _lib.call("ss_krylov_residuals", self._h, int(nb), _lib.stream_ptr(self.device), _lib.ptr(out))
        return out

    def history(self, mode: int, count: int) -> list:
        count = int(min(count, self.hist_cap))
        out = np.zeros(max(count, 1))
        if count:
            _lib.call("ss_krylov_history", self._h, int(mode), count, _lib.ptr(out))
        return [float(v) for v in out[:count]]

    def done_ticks(self, nb: int) -> np.ndarray:
        """Tick at which each mode of the last solve finished (ss_krylov_done_ticks)."""
        out = np.zeros(nb, dtype=np.int64)
        _lib.call("ss_krylov_done_ticks", self._h, int(nb), _lib.ptr(out, C.c_int64))
        return out

    def last_stats(self):
        t, l = C.c_int64(), C.c_int64()
        _lib.call("ss_krylov_last_stats", self._h, C.byref(t), C.byref(l))
        return int(t.value), int(l.value)

    def load_rhs(self, rhs):
        """Copy (nb, ld) device right-hand sides into the workspace."""
        _lib.call("ss_krylov_copy", self._h, int(rhs.shape[0]), 0, _lib.dptr(rhs), int(rhs.shape[1]),
                  _lib.stream_ptr(self.device))

    def profile(self, omegas, tol, maxiter, jacobi=True):
        """Instrumented (event-timed, un-graphed) solve of the workspace's RHS: per-kernel ms/bytes/launches."""
        om = np.ascontiguousarray(np.asarray(omegas, dtype=float).reshape(-1))
        ms = np.zeros(5)
        by = np.zeros(5, dtype=np.int64)
        ln = np.zeros(5, dtype=np.int64)
        _lib.call("ss_krylov_profile", self._h, om.size, _lib.ptr(om), float(tol), int(maxiter), int(bool(jacobi)),
                  _lib.stream_ptr(self.device), _lib.ptr(ms), _lib.ptr(by, C.c_int64), _lib.ptr(ln, C.c_int64))
        names = ["spmv", "passA_dot", "passB_update_dot", "passC_update_norm", "passX_xupdate"]
        return {n: dict(ms=float(m), bytes=int(b), launches=int(l)) for n, m, b, l in zip(names, ms, by, ln)}

    def bench_pass(self, nb: int, k: int, which: int = 2, reps: int = 5):
        ms, by = C.c_float(), C.c_int64()
        _lib.call("ss_krylov_bench_pass", self._h, int(nb), int(k), int(which), int(reps),
                  _lib.stream_ptr(self.device), C.byref(ms), C.byref(by))
        return float(ms.value), int(by.value)


def jacobi_precondition(system) -> np.ndarray:
    """Reciprocal-diagonal scaling; 1 where the diagonal is zero (krylov.py:49-60)."""
    from .assembly import ComplexSaddleSystem

    if isinstance(system, ComplexSaddleSystem):
        op = system.operator
        return op.jacobi([system.omega])[0, : op.n].cpu().numpy()
    matrix = getattr(system, "matrix", system)
    ws = KrylovWorkspace.for_csr(matrix, 1, 1, 1, jacobi_from_diag=True)
    try:
        return ws.csr_scale()
    finally:
        ws.close()


def _to_device_rows(vec, ld, device):
    torch = _lib.torch_mod()
    out = torch.zeros((1, ld), dtype=torch.complex128, device=device)
    v = np.ascontiguousarray(np.asarray(vec, dtype=complex).ravel())
    out[0, : v.size] = torch.from_numpy(v).to(device)
    return out


def gmres(matrix, rhs, tol=1e-6, restart=200, maxiter=200_000, scale=None, x0=None):
    """Left-preconditioned restarted GMRES; returns ``(x, iterations, history, converged)`` (krylov.py:63-164)."""
    n = matrix.shape[0]
    ws = KrylovWorkspace.for_csr(matrix, restart, 1, max(1, int(maxiter)), scale=scale)
    try:
        b = _to_device_rows(rhs, ws.ld, ws.device)
        x0d = None if x0 is None else _to_device_rows(x0, ws.ld, ws.device)
        out = ws.solve([0.0], b, x0d, tol, maxiter, jacobi=scale is not None)
        x = out["x"][0, :n].cpu().numpy()
        hist = ws.history(0, int(out["hist_len"][0]))
        return x, int(out["iterations"][0]), hist, bool(out["converged"][0])
    finally:
        ws.close()


def gmres_solve(system, settings: SolverSettings, x0=None):
    """Solve an assembled system or ``(matrix, rhs)``; returns ``(x, SolveReport)`` (krylov.py:171-216)."""
    from .assembly import ComplexSaddleSystem

    jac = settings.preconditioner == "jacobi"
    wall0, cpu0 = time.perf_counter(), time.thread_time()
    if not isinstance(system, (tuple, ComplexSaddleSystem)) and hasattr(system, "matrix") and hasattr(system, "rhs"):
        system = (system.matrix, system.rhs)   # a system assembled by other code (e.g. the reference's CPU path)
    if isinstance(system, tuple):
        matrix, rhs = system
        n = matrix.shape[0]
        ws = KrylovWorkspace.for_csr(matrix, settings.restart, 1, max(1, settings.max_iterations),
                                     jacobi_from_diag=jac)
        try:
            b = _to_device_rows(rhs, ws.ld, ws.device)
            x0d = None if x0 is None else _to_device_rows(x0, ws.ld, ws.device)
            out = ws.solve([0.0], b, x0d, settings.tolerance, settings.max_iterations, jacobi=jac)
            wall, cpu = time.perf_counter() - wall0, time.thread_time() - cpu0
            res = float(ws.residuals(1)[0])
            x = out["x"][0, :n].cpu().numpy()
            hist = ws.history(0, int(out["hist_len"][0]))
        finally:
            ws.close()
    elif isinstance(system, ComplexSaddleSystem):
        op = system.operator
        with op.lock:
            ws = op.krylov(settings.restart, 1, max(1, settings.max_iterations))
            x0d = None if x0 is None else _to_device_rows(x0, ws.ld, ws.device)
            out = ws.solve([system.omega], system._rhs_dev, x0d, settings.tolerance, settings.max_iterations,
                           jacobi=jac)
            wall, cpu = time.perf_counter() - wall0, time.thread_time() - cpu0
            res = float(ws.residuals(1)[0])
            x = out["x"][0, : op.n].cpu().numpy()
            hist = ws.history(0, int(out["hist_len"][0]))
    else:
        raise TypeError("system must be a ComplexSaddleSystem or a (matrix, rhs) tuple")
    report = SolveReport(iterations=int(out["iterations"][0]), residual=res,
                         converged=bool(out["converged"][0] and res <= settings.tolerance),
                         wall_time=wall, cpu_time=cpu, residual_history=hist)
    return x, report


MAX_BATCH = 256   # modes per device batch (ss_krylov_create_*: per-tick mode state lives in smem)


def gmres_batched(batch, settings: SolverSettings, x0=None, keep_history=True):
    """Solve every mode of a :class:`~.assembly.ModeSystemBatch` in one device batch (chunks of
    MAX_BATCH modes beyond that; per-mode results do not depend on the chunking).

    Returns ``(X, reports)`` with ``X`` the (nb, ld) complex128 device solutions.
    """
    op = batch.operator
    nb = batch.nb
    if nb > MAX_BATCH:
        from .assembly import ModeSystemBatch

        torch = _lib.torch_mod()
        xs, reps = [], []
        for s in range(0, nb, MAX_BATCH):
            sl = slice(s, min(nb, s + MAX_BATCH))
            per_mode = lambda v: None if v is None else v[sl]  # noqa: E731
            sub = ModeSystemBatch(op, batch.omegas[sl], batch.rhs[sl], per_mode(batch.g), per_mode(batch.dirichlet),
                                  per_mode(getattr(batch, "loads", None)))
            X, r = gmres_batched(sub, settings, None if x0 is None else x0[sl], keep_history)
            xs.append(X)
            reps.extend(r)
        return torch.cat(xs, dim=0), reps
    jac = settings.preconditioner == "jacobi"
    hist_cap = max(1, settings.max_iterations)
    k = concurrent_groups(op.n, nb)
    with op.lock:
        wall0, cpu0 = time.perf_counter(), time.thread_time()
        if k == 1:
            ws = op.krylov(settings.restart, nb, hist_cap)
            out = ws.solve(batch.omegas, batch.rhs, x0, settings.tolerance, settings.max_iterations, jacobi=jac)
            frac = _tick_fractions(ws.done_ticks(nb))
            res = ws.residuals(nb)
            hists = [ws.history(b, int(out["hist_len"][b])) if keep_history else [] for b in range(nb)]
            X, iters, conv = out["x"], out["iterations"], out["converged"]
        else:
            X, iters, conv, res, hists, frac = _solve_concurrent(op, batch, x0, settings, jac, hist_cap, keep_history,
                                                                 k)
        wall, cpu = time.perf_counter() - wall0, time.thread_time() - cpu0
    reports = []
    for b in range(nb):
        # a mode's wall/cpu time: the batch's, scaled by the share of its ticks (the device finishes
        # modes at different ticks; the reference times each mode's own solve, krylov.py:194-202)
        reports.append(SolveReport(iterations=int(iters[b]), residual=float(res[b]),
                                   converged=bool(conv[b] and res[b] <= settings.tolerance),
                                   wall_time=wall * frac[b], cpu_time=cpu * frac[b], residual_history=hists[b]))
    return X, reports


def _tick_fractions(done_ticks) -> np.ndarray:
    t = np.asarray(done_ticks, dtype=float)
    top = t.max() if t.size else 0.0
    return t / top if top > 0 else np.ones_like(t)


def concurrent_groups(n: int, nb: int) -> int:
    """Sub-batches run concurrently (own workspace, CUDA stream and host thread) for small systems:
    each tick kernel of a small system leaves SMs idle in its latency tails, which the other
    sub-batches fill (measured: 17 modes at n = 8 782 +24 % with 4 groups; 9 modes at n = 9 103
    +4 %).  Per-mode results are bitwise independent of the grouping (batch invariance)."""
    if n >= 200_000:
        return 1
    if os.environ.get("SS_FUSED", "0") not in ("", "0"):
        return 1   # persistent cooperative tick kernels occupy every SM: never two at once
    k = max(1, min(4, nb // 3))   # sub-batches of >= 3 modes (config 1: 4 groups of 2-3 measured -13 %)
    env = os.environ.get("SS_CONCURRENT_GROUPS")   # A/B knob (tools/c1_public_ab.py)
    return max(1, min(nb, int(env))) if env else k


def _solve_concurrent(op, batch, x0, settings, jac, hist_cap, keep_history, k):
    import threading

    torch = _lib.torch_mod()
    nb = batch.nb
    groups = [list(range(g, nb, k)) for g in range(k)]
    wss = [op.krylov(settings.restart, len(g), hist_cap, slot=i) for i, g in enumerate(groups)]
    rhs = [batch.rhs[g].contiguous() for g in groups]
    x0s = [None if x0 is None else x0[g].contiguous() for g in groups]
    torch.cuda.synchronize(op.device)
    streams = [torch.cuda.Stream(op.device) for _ in groups]
    outs, errs = [None] * k, [None] * k

    def run(i):
        try:
            with torch.cuda.stream(streams[i]):
                o = wss[i].solve(batch.omegas[groups[i]], rhs[i], x0s[i], settings.tolerance,
                                 settings.max_iterations, jacobi=jac)
                res = wss[i].residuals(len(groups[i]))
                h = [wss[i].history(b, int(o["hist_len"][b])) if keep_history else [] for b in range(len(groups[i]))]
                torch.cuda.current_stream().synchronize()
                outs[i] = (o, res, h, wss[i].done_ticks(len(groups[i])))
        except BaseException as exc:   # re-raised in the caller's thread
            errs[i] = exc

    threads = [threading.Thread(target=run, args=(i,)) for i in range(k)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    for e in errs:
        if e is not None:
            raise e
    X = torch.empty((nb, op.ld), dtype=torch.complex128, device=op.device)
    iters = np.zeros(nb, dtype=np.int64)
    conv = np.zeros(nb, dtype=bool)
    res = np.zeros(nb)
    hists = [None] * nb
    ticks = np.zeros(nb)
    for i, g in enumerate(groups):
        o, r, h, t = outs[i]
        ticks[g] = t
        X[g] = o["x"]
        iters[g] = o["iterations"]
        conv[g] = o["converged"]
        res[g] = r
        for j, b in enumerate(g):
            hists[b] = h[j]
    return X, iters, conv, res, hists, _tick_fractions(ticks)
