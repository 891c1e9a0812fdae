"""Drop-in assembly API backed by the device operator (reference `assembly.py`).

Same names, signatures, argument meaning and errors as `pkg/src/spectralstokes/assembly.py`:
``FluidProps`` (24-37), ``ShapeSet``/``reference_shapes`` (40-128), ``boundary_traction_load``
(249-262), ``ComplexSaddleSystem`` (312-379) and ``assemble_mode_system`` (403-494).

What differs is where the work happens.  The reference re-assembles the whole complex matrix with
scipy for every mode (spectral.py:280).  Here a mesh + fluid pair owns ONE device operator
(:class:`SaddleOperator`): the symbolic pattern and element maps are built once on the host
(`csrc/pattern.cpp`), the real S', M', D values once on the device (`csrc/assemble.cu`), and a
mode is just its frequency plus a right-hand side assembled on the device.  ``system.matrix`` is
materialised lazily as a scipy CSR (bit-identical pattern) only for callers that ask for it.
"""

from __future__ import annotations

import ctypes as C
import threading
import weakref
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from . import _lib
from .errors import MeshError
from .mesh import QuadraticMesh

__all__ = [
    "FluidProps", "ShapeSet", "reference_shapes", "boundary_traction_load", "ComplexSaddleSystem",
    "ModeSystemBatch", "SaddleOperator", "assemble_mode_system", "assemble_mode_systems", "get_operator",
    "dirichlet_values_from_patches", "constrained_velocity_nodes",
]


@dataclass
class FluidProps:
    """Newtonian fluid constants (assembly.py:24-37)."""

    density: float
    viscosity: float

    def __post_init__(self):
        if self.density <= 0 or self.viscosity <= 0:
            raise ValueError("density and viscosity must be positive")

    @property
    def kinematic_viscosity(self) -> float:
        return self.viscosity / self.density


@dataclass
class ShapeSet:
    """Reference-simplex shape values, gradients and quadrature weights (assembly.py:40-48)."""

    points: np.ndarray
    weights: np.ndarray
    vel_values: np.ndarray
    vel_grads: np.ndarray
    pres_values: np.ndarray


def _rule(dim):
    if dim == 2:
        pairs = ((0.445948490915965, 0.223381589678011), (0.091576213509771, 0.109951743655322))
        bary, w = [], []
        for a, wt in pairs:
            for i in range(3):
                b = [a, a, a]
                b[i] = 1 - 2 * a
                bary.append(b)
                w.append(0.5 * wt)
        return np.array([(b[1], b[2]) for b in bary]), np.array(w)
    root = np.sqrt(5.0 / 14.0)
    hi, lo = (1.0 + root) / 4.0, (1.0 - root) / 4.0
    bary, w = [[0.25] * 4], [-74.0 / 5625.0]
    for i in range(4):
        b = [1.0 / 14.0] * 4
        b[i] = 11.0 / 14.0
        bary.append(b)
        w.append(343.0 / 45000.0)
    for i in range(4):
        for j in range(i + 1, 4):
            b = [lo] * 4
            b[i] = b[j] = hi
            bary.append(b)
            w.append(56.0 / 2250.0)
    return np.array([b[1:] for b in bary]), np.array(w)


def reference_shapes(dim: int, quadrature_order: int = 4) -> ShapeSet:
    """P2 velocity / P1 pressure bases at the degree-4 rule (assembly.py:115-128)."""
    if dim not in (2, 3):
        raise ValueError(f"unsupported dimension {dim}")
    if quadrature_order != 4:
        raise ValueError(f"unsupported quadrature order {quadrature_order} (only 4)")
    pts, w = _rule(dim)
    lam = np.column_stack([1.0 - pts.sum(axis=1), pts])
    dlam = np.vstack([-np.ones(dim), np.eye(dim)])
    edges = ((0, 1), (1, 2), (2, 0)) if dim == 2 else ((0, 1), (1, 2), (0, 2), (0, 3), (1, 3), (2, 3))
    nb = dim + 1 + len(edges)
    vals = np.empty((pts.shape[0], nb))
    grads = np.empty((pts.shape[0], nb, dim))
    for v in range(dim + 1):
        vals[:, v] = lam[:, v] * (2.0 * lam[:, v] - 1.0)
        grads[:, v, :] = (4.0 * lam[:, v] - 1.0)[:, None] * dlam[v]
    for e, (i, j) in enumerate(edges):
        vals[:, dim + 1 + e] = 4.0 * lam[:, i] * lam[:, j]
        grads[:, dim + 1 + e, :] = 4.0 * (lam[:, i][:, None] * dlam[j] + lam[:, j][:, None] * dlam[i])
    return ShapeSet(pts, w, vals, grads, lam)


# ------------------------------------------------------------------------------------------------
# Boundary data helpers (host; boundary faces only)
# ------------------------------------------------------------------------------------------------

def constrained_velocity_nodes(qmesh) -> np.ndarray:
    """Velocity nodes on dirichlet/wall patches (assembly.py:392-400)."""
    parts = [p.face_conn.ravel() for p in qmesh.boundary_patches.values() if p.kind in ("dirichlet", "wall")]
    return np.unique(np.concatenate(parts)) if parts else np.empty(0, dtype=np.int64)


def dirichlet_values_from_patches(qmesh, patch_values: dict) -> np.ndarray:
    """Uniform per-patch velocity vectors -> nodal array; later patches win (assembly.py:382-389)."""
    g = np.zeros((qmesh.n_velocity_nodes, qmesh.dim), dtype=complex)
    for name, vec in patch_values.items():
        g[np.unique(qmesh.boundary_patches[name].face_conn)] = np.asarray(vec, dtype=complex)
    return g


def boundary_traction_load(qmesh, patch: str, h_mode) -> np.ndarray:
    """Consistent nodal load of traction data on a Neumann patch (assembly.py:249-262).

    Computed by the library's host routine ``ss_surface_load`` (boundary faces only).
    """
    try:
        pdata = qmesh.boundary_patches[patch]
    except KeyError:
        raise MeshError(f"unknown boundary patch '{patch}'") from None
    if pdata.kind != "neumann":
        raise MeshError(f"patch '{patch}' is {pdata.kind}, not neumann")
    dim = qmesh.dim
    conn = np.ascontiguousarray(pdata.face_conn, dtype=np.int64)
    nf = conn.shape[0]
    load = np.zeros((qmesh.n_velocity_nodes, dim), dtype=complex)
    if nf == 0:
        return load
    h = np.ascontiguousarray(np.asarray(h_mode, dtype=complex))
    if h.shape == (dim,):
        kind = 0
    elif h.shape == (nf, dim):
        kind = 1
    elif h.shape == (qmesh.n_velocity_nodes, dim):
        kind = 2
    else:
        raise ValueError(f"traction data shape {h.shape} does not match patch or mesh")
    nodes = np.ascontiguousarray(qmesh.nodes, dtype=float)
    _lib.call("ss_surface_load", dim, qmesh.n_velocity_nodes, _lib.ptr(nodes), nf,
              _lib.ptr(conn, C.c_int64), kind, _lib.ptr(h.view(np.float64)), _lib.ptr(load.view(np.float64)))
    return load


# ------------------------------------------------------------------------------------------------
# Device operator
# ------------------------------------------------------------------------------------------------

class SaddleOperator:
    """One mesh + fluid on one GPU: pattern, element maps and assembled S', M', D.

    ``A(w) = [[S' (x) I + i w M' (x) I, D], [D^T, 0]]`` reduced to the free DOFs of the
    reference numbering (assembly.py:424-479).  The operator is frequency-free; every entry
    point takes per-mode frequencies.
    """

    def __init__(self, qmesh, props: FluidProps, device=None):
        torch = _lib.torch_mod()
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self.dim = qmesh.dim
        self.n_vel_nodes = qmesh.n_velocity_nodes
        self.n_vertices = qmesh.n_vertices
        self.props = props
        fixed = constrained_velocity_nodes(qmesh)
        mask = np.zeros(self.n_vel_nodes, dtype=np.uint8)
        mask[fixed] = 1
        self.fixed_nodes = fixed
        self.fixed_mask = mask.astype(bool)
        neumann = [p for p in qmesh.boundary_patches.values() if p.kind == "neumann"]
        self.pinned = not any(p.faces.size for p in neumann)
        conn = np.ascontiguousarray(qmesh.vel_conn, dtype=np.int64)
        h = C.c_void_p()
        with torch.cuda.device(self.device):
            _lib.call("ss_pattern_create", self.dim, self.n_vel_nodes, self.n_vertices, conn.shape[0],
                      _lib.ptr(conn, C.c_int64), _lib.ptr(mask, C.c_uint8), int(self.pinned),
                      self.device.index, C.byref(h))
        self._h = h
        self._finalizer = weakref.finalize(self, _lib.load().ss_pattern_destroy, h)
        info = np.zeros(16, dtype=np.int64)
        _lib.call("ss_pattern_info", h, _lib.ptr(info, C.c_int64))
        self.info = info
        self.n = int(info[0])
        self.nnz = int(info[1])
        self.ld = (self.n + 31) // 32 * 32
        self.n_free_nodes, self.n_free_pressures = int(info[2]), int(info[3])
        self.n_colors = int(info[7])
        verts = np.ascontiguousarray(qmesh.nodes[: self.n_vertices], dtype=float)
        with torch.cuda.device(self.device):
            _lib.call("ss_assemble", h, _lib.ptr(verts), float(props.density), float(props.viscosity),
                      _lib.stream_ptr(self.device))
        self._pattern = None
        self._dof = None
        self._krylov = {}
        # Cached Krylov workspaces hold device RHS/X/basis buffers and a native graph cache: one
        # host thread at a time per operator (the reference's solve_modes(workers>1) thread pool,
        # spectral.py:300-305, may call gmres_solve concurrently on systems of one mesh).
        self.lock = threading.RLock()

    @property
    def handle(self):
        return self._h

    # -- host views ------------------------------------------------------------------------------
    def pattern(self):
        """(indptr, indices) int32, bit-identical to the reference's reduced CSR."""
        if self._pattern is None:
            ip = np.zeros(self.n + 1, dtype=np.int32)
            ix = np.zeros(self.nnz, dtype=np.int32)
            _lib.call("ss_pattern_export", self._h, _lib.ptr(ip, C.c_int32), _lib.ptr(ix, C.c_int32))
            self._pattern = (ip, ix)
        return self._pattern

    def pattern_rows(self, rows):
        """Column indices of selected reduced rows (list of int32 arrays), bit-exact like pattern()."""
        rows = np.ascontiguousarray(np.asarray(rows, dtype=np.int64))
        counts = np.zeros(rows.size, dtype=np.int64)
        _lib.call("ss_pattern_export_rows", self._h, rows.size, _lib.ptr(rows, C.c_int64), _lib.ptr(counts, C.c_int64),
                  None, 0)
        idx = np.zeros(max(1, int(counts.sum())), dtype=np.int32)
        _lib.call("ss_pattern_export_rows", self._h, rows.size, _lib.ptr(rows, C.c_int64), _lib.ptr(counts, C.c_int64),
                  _lib.ptr(idx, C.c_int32), idx.size)
        return np.split(idx[: int(counts.sum())], np.cumsum(counts)[:-1])

    def constrained_rows(self, omega: float):
        """scipy CSR of a_full[fixed_idx] at ``omega`` (assembly.py:471-476,491)."""
        import scipy.sparse as sp

        info = np.zeros(2, dtype=np.int64)
        _lib.call("ss_constrained_rows", self._h, float(omega), _lib.ptr(info, C.c_int64), None, None, None)
        nrows, nnz = int(info[0]), int(info[1])
        ip = np.zeros(nrows + 1, dtype=np.int64)
        ix = np.zeros(max(1, nnz), dtype=np.int32)
        data = np.zeros(max(1, nnz), dtype=complex)
        _lib.call("ss_constrained_rows", self._h, float(omega), _lib.ptr(info, C.c_int64), _lib.ptr(ip, C.c_int64),
                  _lib.ptr(ix, C.c_int32), _lib.ptr(data.view(np.float64)))
        ncols = self.n_vel_nodes * self.dim + self.n_vertices
        return sp.csr_matrix((data[:nnz], ix[:nnz], ip), shape=(nrows, ncols))

    def dof_maps(self):
        if self._dof is None:
            vd = np.zeros((self.n_vel_nodes, self.dim), dtype=np.int64)
            pd = np.zeros(self.n_vertices, dtype=np.int64)
            _lib.call("ss_pattern_dof_maps", self._h, _lib.ptr(vd, C.c_int64), _lib.ptr(pd, C.c_int64))
            self._dof = (vd, pd)
        return self._dof

    def values(self, omega: float):
        """Reduced-matrix values at ``omega`` in pattern order (device tensor, complex128)."""
        torch = _lib.torch_mod()
        out = torch.empty(self.nnz, dtype=torch.complex128, device=self.device)
        _lib.call("ss_export_values", self._h, float(omega), _lib.dptr(out), _lib.stream_ptr(self.device))
        return out

    def scipy_matrix(self, omega: float):
        import scipy.sparse as sp

        ip, ix = self.pattern()
        data = self.values(omega).cpu().numpy()
        return sp.csr_matrix((data, ix, ip), shape=(self.n, self.n))

    # -- device compute --------------------------------------------------------------------------
    def _omegas(self, omegas):
        torch = _lib.torch_mod()
        return torch.as_tensor(np.asarray(omegas, dtype=float).reshape(-1), device=self.device)

    def rhs(self, omegas, loads=None, gs=None):
        """Right-hand sides (nb, ld) complex128 on the device (assembly.py:432-478)."""
        torch = _lib.torch_mod()
        om = self._omegas(omegas)
        nb = om.numel()
        out = torch.empty((nb, self.ld), dtype=torch.complex128, device=self.device)
        ld_ = None if loads is None else loads.contiguous()
        g_ = None if gs is None else gs.contiguous()
        _lib.call("ss_rhs_batched", self._h, nb, _lib.dptr(om), None if ld_ is None else _lib.dptr(ld_),
                  None if g_ is None else _lib.dptr(g_), _lib.dptr(out), self.ld, _lib.stream_ptr(self.device))
        return out

    def spmv(self, omegas, x, jacobi=False, out=None):
        """Mode-batched Y[b] = s_b .* (A(w_b) X[b]); x (nb, ld) complex128 device tensor."""
        torch = _lib.torch_mod()
        om = self._omegas(omegas)
        nb = om.numel()
        if x.shape != (nb, self.ld) or x.dtype != torch.complex128:
            raise ValueError(f"x must be ({nb}, {self.ld}) complex128")
        y = torch.zeros_like(x) if out is None else out
        _lib.call("ss_spmv_batched", self._h, nb, _lib.dptr(om), _lib.dptr(x), _lib.dptr(y), self.ld,
                  int(bool(jacobi)), _lib.stream_ptr(self.device))
        return y

    def residual_norms(self, omegas, rhs, x):
        """||b - A x|| / ||b|| per mode (device kernels, fixed-order reduction)."""
        om = self._omegas(omegas)
        out = np.zeros(om.numel())
        _lib.call("ss_residual_norms", self._h, om.numel(), _lib.dptr(om), _lib.dptr(rhs), _lib.dptr(x), self.ld,
                  _lib.ptr(out), _lib.stream_ptr(self.device))
        return out

    def spmv_interleaved(self, omegas, x_int, jacobi=False, out=None):
        """Mode-interleaved SpMV (the GMRES tick's kernel): x_int (ld, nb) row-major, returns (nb, ld)."""
        torch = _lib.torch_mod()
        om = self._omegas(omegas)
        nb = om.numel()
        if tuple(x_int.shape) != (self.ld, nb) or x_int.dtype != torch.complex128:
            raise ValueError(f"x_int must be ({self.ld}, {nb}) complex128")
        y = torch.zeros((nb, self.ld), dtype=torch.complex128, device=self.device) if out is None else out
        _lib.call("ss_spmv_batched_interleaved", self._h, nb, _lib.dptr(om), _lib.dptr(x_int.contiguous()),
                  _lib.dptr(y), self.ld, int(bool(jacobi)), _lib.stream_ptr(self.device))
        return y

    def spmv_bytes(self, nb: int) -> int:
        return int(_lib.load().ss_spmv_bytes(self._h, nb))

    def jacobi(self, omegas):
        torch = _lib.torch_mod()
        om = self._omegas(omegas)
        out = torch.empty((om.numel(), self.ld), dtype=torch.complex128, device=self.device)
        _lib.call("ss_jacobi", self._h, om.numel(), _lib.dptr(om), _lib.dptr(out), self.ld,
                  _lib.stream_ptr(self.device))
        return out

    def expand(self, x, gs=None):
        """Reduced (nb, ld) -> nodal velocity (nb, n_vn, dim) and pressure (nb, n_vert)."""
        torch = _lib.torch_mod()
        nb = x.shape[0]
        u = torch.empty((nb, self.n_vel_nodes, self.dim), dtype=torch.complex128, device=self.device)
        p = torch.empty((nb, self.n_vertices), dtype=torch.complex128, device=self.device)
        _lib.call("ss_expand", self._h, nb, _lib.dptr(x), self.ld, None if gs is None else _lib.dptr(gs.contiguous()),
                  _lib.dptr(u), _lib.dptr(p), _lib.stream_ptr(self.device))
        return u, p

    def krylov(self, restart: int, nb: int, hist_cap: int, slot: int = 0):
        """Cached batched-GMRES workspace with capacity >= nb modes (``slot`` > 0: the extra
        workspaces of concurrently solved sub-batches, krylov.concurrent_groups)."""
        from .krylov import KrylovWorkspace

        key = restart if slot == 0 else (restart, slot)
        ws = self._krylov.get(key)
        if ws is None or ws.max_batch < nb or ws.hist_cap < hist_cap:
            if ws is not None:
                ws.close()
            torch = _lib.torch_mod()
            need = self.workspace_bytes(restart, nb, hist_cap)
            free, _ = torch.cuda.mem_get_info(self.device)
            if need > free:
                from .errors import DeviceError

                raise DeviceError(f"Krylov workspace for {nb} mode(s) at restart {restart} needs {need / 2**30:.1f} GiB; "
                                  f"{free / 2**30:.1f} GiB of device memory is free (fewer modes per batch, a smaller "
                                  f"restart, or free other workspaces: SaddleOperator.release_workspaces)")
            ws = KrylovWorkspace.for_operator(self, restart, nb, hist_cap)
            self._krylov[key] = ws
        return ws

    def release_workspaces(self):
        """Free every cached Krylov workspace (basis, Hessenberg, graphs) of this operator."""
        with self.lock:
            for ws in self._krylov.values():
                ws.close()
            self._krylov.clear()

    def workspace_bytes(self, restart: int, nb: int, hist_cap: int) -> int:
        """Device bytes of a Krylov workspace for ``nb`` modes (mirrors krylov_common_init and
        ss_krylov_create_saddle: basis, W/P/X/RHS, Hessenberg, Givens, partials, history)."""
        ld = self.ld
        jcap = restart + 1
        seg = min(6144, max(256, ((ld + 15) // 16 + 31) // 32 * 32))   # krylov_common_init segment rows
        nseg = -(-ld // seg)
        nsb = -(-self.n_free_nodes // 128) + -(-self.n_free_pressures // 32)
        per_mode = 16 * (jcap * ld + 4 * ld + restart * jcap + 4 * jcap + 2 * restart + nseg * jcap + nsb) \
            + 8 * (jcap + max(1, hist_cap)) + 32 + 96
        return nb * per_mode + 4096

    def max_batch(self, restart: int, hist_cap: int = 200_000) -> int:
        """Modes whose Krylov workspaces fit this GPU now: free HBM minus a reserve (1 GiB + 2 % of
        the device), divided by the exact per-mode workspace size."""
        torch = _lib.torch_mod()
        free, total = torch.cuda.mem_get_info(self.device)
        reserve = (1 << 30) + total // 50
        per_mode = self.workspace_bytes(restart, 1, hist_cap)
        return max(1, min(256, int((free - reserve) // per_mode)))   # 256: krylov.MAX_BATCH


_OP_CACHE: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()


def get_operator(qmesh, props: FluidProps, device=None) -> SaddleOperator:
    """Per-(mesh, fluid, device) cached operator."""
    torch = _lib.torch_mod()
    dev = torch.cuda.current_device() if device is None else int(device)
    try:
        per_mesh = _OP_CACHE.setdefault(qmesh, {})
    except TypeError:
        per_mesh = {}
    key = (float(props.density), float(props.viscosity), dev)
    op = per_mesh.get(key)
    if op is None:
        op = SaddleOperator(qmesh, props, dev)
        per_mesh[key] = op
    return op


# ------------------------------------------------------------------------------------------------
# Mode systems
# ------------------------------------------------------------------------------------------------

def _nodal_dirichlet(qmesh, g_mode):
    n_vn, dim = qmesh.n_velocity_nodes, qmesh.dim
    if g_mode is None:
        return None
    if isinstance(g_mode, dict):
        return dirichlet_values_from_patches(qmesh, g_mode)
    g = np.asarray(g_mode, dtype=complex)
    if g.shape != (n_vn, dim):
        raise ValueError(f"g_mode shape {g.shape} != ({n_vn}, {dim})")
    return g


def _check_dirichlet(op: SaddleOperator, g):
    if g is not None and np.any(g[~op.fixed_mask] != 0):
        raise ValueError("g_mode has nonzero values on nodes that are not Dirichlet-constrained")


def _traction_loads(qmesh, h_mode):
    load = np.zeros((qmesh.n_velocity_nodes, qmesh.dim), dtype=complex)
    for name, data in (h_mode or {}).items():
        load += boundary_traction_load(qmesh, name, data)
    return load


@dataclass
class ModeSystemBatch:
    """nb mode systems sharing one operator; everything device-resident."""

    operator: SaddleOperator
    omegas: np.ndarray
    rhs: object              # (nb, ld) complex128 device tensor
    g: object                # (nb, n_vn, dim) complex128 device tensor or None
    dirichlet: list          # per-mode host nodal Dirichlet arrays (None = zero)
    loads: list = None       # per-mode host traction loads (None = zero)

    @property
    def nb(self):
        return len(self.omegas)


def assemble_mode_systems(qmesh, props: FluidProps, omegas, g_modes=None, h_modes=None, operator=None,
                          g_device=None):
    """Batched ``assemble_mode_system`` for many modes at once (one device RHS launch).

    ``g_device`` optionally supplies the nodal Dirichlet data of all modes as a device tensor
    (nb, n_vel_nodes, dim) complex128 that the caller guarantees is zero off constrained nodes
    (the zero-copy path used by the end-to-end benchmark); it replaces ``g_modes``.
    """
    torch = _lib.torch_mod()
    omegas = np.asarray(omegas, dtype=float).reshape(-1)
    if np.any(omegas < 0):
        raise ValueError("omega must be non-negative")
    nb = omegas.size
    op = operator or get_operator(qmesh, props)
    if g_device is not None:
        if tuple(g_device.shape) != (nb, qmesh.n_velocity_nodes, qmesh.dim) or g_device.dtype != torch.complex128:
            raise ValueError("g_device must be (nb, n_velocity_nodes, dim) complex128")
        loads = None
        if h_modes is not None and any(h for h in h_modes):
            host = np.stack([_traction_loads(qmesh, h) for h in h_modes])
            loads = torch.from_numpy(host).to(op.device)
        return ModeSystemBatch(op, omegas, op.rhs(omegas, loads, g_device), g_device, [None] * nb)
    gl = [None] * nb if g_modes is None else [_nodal_dirichlet(qmesh, g) for g in g_modes]
    hl = [None] * nb if h_modes is None else list(h_modes)
    for g in gl:
        _check_dirichlet(op, g)
    loads = None
    load_host = [None] * nb
    if any(h for h in hl):
        host = np.stack([_traction_loads(qmesh, h) for h in hl])
        load_host = list(host)
        loads = torch.from_numpy(host).to(op.device)
    gdev = None
    if any(g is not None for g in gl):
        host = np.stack([np.zeros((qmesh.n_velocity_nodes, qmesh.dim), complex) if g is None else g for g in gl])
        gdev = torch.from_numpy(host).to(op.device)
    rhs = op.rhs(omegas, loads, gdev)
    return ModeSystemBatch(op, omegas, rhs, gdev, gl, load_host)


class ComplexSaddleSystem:
    """Reduced complex saddle-point system of one mode (assembly.py:312-379), device-backed."""

    def __init__(self, operator: SaddleOperator, omega: float, rhs_dev, g_dev, g_host, load_host=None):
        self.operator = operator
        self.omega = float(omega)
        self._rhs_dev = rhs_dev            # (1, ld)
        self._g_dev = g_dev                # (1, n_vn, dim) or None
        n_vn, dim = operator.n_vel_nodes, operator.dim
        store = np.zeros((n_vn, dim), dtype=complex)
        if g_host is not None:
            store[operator.fixed_nodes] = g_host[operator.fixed_nodes]
        self.dirichlet_values = store
        self.vel_dof, self.pres_dof = operator.dof_maps()
        self.pinned_pressure = operator.pinned
        self._load = load_host
        self._rhs = None
        self._matrix = None
        self._constrained = None

    @property
    def rhs(self) -> np.ndarray:
        if self._rhs is None:
            self._rhs = self._rhs_dev[0, : self.operator.n].cpu().numpy()
        return self._rhs

    @property
    def matrix(self):
        """scipy CSR of the reduced matrix (materialised on demand; pattern bit-exact)."""
        if self._matrix is None:
            self._matrix = self.operator.scipy_matrix(self.omega)
        return self._matrix

    @property
    def n_dofs(self) -> int:
        return self.operator.n

    @property
    def n_velocity_dofs(self) -> int:
        return int((self.vel_dof >= 0).sum())

    @property
    def n_pressure_dofs(self) -> int:
        return int((self.pres_dof >= 0).sum())

    def expand(self, x: np.ndarray):
        """Reduced solution -> nodal velocity and pressure (assembly.py:338-346)."""
        u = self.dirichlet_values.astype(complex).copy()
        m = self.vel_dof >= 0
        u[m] = x[self.vel_dof[m]]
        p = np.zeros(self.pres_dof.shape[0], dtype=complex)
        pm = self.pres_dof >= 0
        p[pm] = x[self.pres_dof[pm]]
        return u, p

    def flatten(self, u: np.ndarray, p: np.ndarray) -> np.ndarray:
        """Nodal fields -> reduced vector (assembly.py:348-355)."""
        x = np.zeros(self.n_dofs, dtype=complex)
        m = self.vel_dof >= 0
        x[self.vel_dof[m]] = u[m]
        pm = self.pres_dof >= 0
        x[self.pres_dof[pm]] = p[pm]
        return x

    def residual_norm(self, x: np.ndarray) -> float:
        """True relative residual of the reduced system at ``x`` (assembly.py:357-362), on device."""
        torch = _lib.torch_mod()
        op = self.operator
        xd = torch.zeros((1, op.ld), dtype=torch.complex128, device=op.device)
        xd[0, : op.n] = torch.from_numpy(np.ascontiguousarray(x, dtype=complex)).to(op.device)
        return float(op.residual_norms([self.omega], self._rhs_dev, xd)[0])

    @property
    def constrained_rows(self):
        """a_full[fixed_idx] as scipy CSR (assembly.py:322,491), device-assembled."""
        if self._constrained is None:
            self._constrained = self.operator.constrained_rows(self.omega)
        return self._constrained

    @property
    def constrained_rhs(self) -> np.ndarray:
        """rhs_full[fixed_idx] (assembly.py:323,492): traction load at fixed DOFs, 0 for a pinned pressure."""
        op = self.operator
        fixed_idx = (op.fixed_nodes[:, None] * op.dim + np.arange(op.dim)).ravel()
        load = np.zeros(op.n_vel_nodes * op.dim, dtype=complex) if self._load is None else self._load.ravel()
        out = load[fixed_idx]
        if op.pinned:
            out = np.concatenate([out, [0.0]])
        return np.asarray(out, dtype=complex)

    def reaction_forces(self, x: np.ndarray) -> np.ndarray:
        """Nodal forces on constrained velocity DOFs (assembly.py:364-367)."""
        u, p = self.expand(x)
        full = np.concatenate([u.ravel(), p])
        return np.asarray(self.constrained_rows @ full - self.constrained_rhs)

    def export_matrix(self, path) -> None:
        """Coordinate-list text dump ``row col re im`` (assembly.py:373-379)."""
        coo = self.matrix.tocoo()
        with open(Path(path), "w") as fh:
            fh.write(f"# {coo.shape[0]} {coo.shape[1]} {coo.nnz}\n")
            for r, c, v in zip(coo.row, coo.col, coo.data):
                fh.write(f"{r} {c} {v.real:.17g} {v.imag:.17g}\n")


def assemble_mode_system(qmesh, props: FluidProps, omega: float, g_mode=None, h_mode=None,
                         viscous_form: str = "full") -> ComplexSaddleSystem:
    """Assemble the complex system for one frequency (assembly.py:403-494)."""
    if omega < 0:
        raise ValueError("omega must be non-negative")
    if viscous_form not in ("full", "symmetric"):
        raise ValueError(f"unknown viscous form '{viscous_form}'")
    if viscous_form == "symmetric":
        raise NotImplementedError("the symmetric viscous form is outside the B200 hot path (SURVEY.md §8a row 5)")
    batch = assemble_mode_systems(qmesh, props, [omega], None if g_mode is None else [g_mode],
                                  None if h_mode is None else [h_mode])
    return ComplexSaddleSystem(batch.operator, omega, batch.rhs, batch.g, batch.dirichlet[0],
                               None if batch.loads is None else batch.loads[0])
