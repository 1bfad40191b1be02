"""Thin ctypes binding of libfde (include/fde.h): argument marshalling only.

Every step of the method runs in the CUDA kernels of libfde.so; this module
only converts Python / torch arguments into pointers and sizes.  There is no
fallback: if the library cannot be loaded, or no CUDA device is visible,
the calls raise.

Vector convention: a block of `nrhs` vectors of length n in the paper's X
ordering is a torch float64 CUDA tensor of shape (nrhs, n)
(row-major = column-major n x nrhs with ld = n).
"""
from __future__ import annotations

import ctypes
import os
from typing import List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libfde.so")
_lib = None

# error codes (include/fde.h)
ERRORS = {
    -1: "FDE_EINVAL_DOMAIN", -2: "FDE_EINVAL_SIZE", -3: "FDE_EINVAL_PARAM", -4: "FDE_EINVAL_MESH",
    -5: "FDE_EDEGREE", -6: "FDE_EUNSUPPORTED_MESH", -7: "FDE_EDIM", -8: "FDE_ESINGULAR_PIVOT",
    -9: "FDE_EBREAKDOWN", -10: "FDE_EMAXITER", -11: "FDE_ECUDA", -12: "FDE_ENCCL", -13: "FDE_ENOMEM",
    -14: "FDE_ERANK",
}
OP_DENSE, OP_TOEPLITZ = 1, 2
PATH_AUTO, PATH_DENSE, PATH_TOEPLITZ = 0, 1, 2
GMRES, BICGSTAB = 0, 1
MESH_CUSTOM, MESH_UNIFORM = 0, 1

EXPORTED = [
    "fde_create", "fde_destroy", "fde_last_error", "fde_sync", "fde_nccl_unique_id",
    "sem_assemble", "fde_operator_get_info", "fde_operator_dense_paper", "fde_operator_boundary_columns",
    "sem_rhs", "stiffness_matvec", "hmatrix_build", "fde_hmatrix_get_info", "fde_hmatrix_dense_paper",
    "hlu_factor", "fde_hlu_get_info", "fde_hlu_dense_internal", "precond_apply", "solve", "fde_solve",
    "fde_free_operator", "fde_free_hmatrix", "fde_free_hlu", "fde_profile", "fde_profile_collect",
    "fde_launch_count", "fde_shard_rows", "fde_debug_hlu_mode", "fde_debug_pool_bytes",
    "fde_operator_wait", "fde_hmatrix_wait", "fde_create_virtual_rank", "fde_operator_rows_internal",
    "fde_shard_matvec", "fde_debug_compact_gather", "hmatrix_build_partition", "fde_debug_truncate",
    "fde_debug_trunc_profile", "fde_debug_comm_selftest",
]
PARTITION_INTERLEAVED, PARTITION_PAPER = 0, 1


class FdeError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code
        self.name = ERRORS.get(code, str(code))


class Problem(ctypes.Structure):
    _fields_ = [("a", ctypes.c_double), ("b", ctypes.c_double), ("alpha", ctypes.c_double),
                ("theta", ctypes.c_double), ("rho", ctypes.c_double), ("c1", ctypes.c_double),
                ("c2", ctypes.c_double)]


class Mesh(ctypes.Structure):
    _fields_ = [("N", ctypes.c_int32), ("nodes", ctypes.POINTER(ctypes.c_double)), ("P", ctypes.c_int32),
                ("kind", ctypes.c_int32)]


class Forcing(ctypes.Structure):
    _fields_ = [("nleg", ctypes.c_int32), ("leg", ctypes.POINTER(ctypes.c_double)),
                ("nterm", ctypes.c_int32), ("side", ctypes.POINTER(ctypes.c_int32)),
                ("power", ctypes.POINTER(ctypes.c_double)), ("coef", ctypes.POINTER(ctypes.c_double))]


class OperatorInfo(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("N", ctypes.c_int32), ("P", ctypes.c_int32),
                ("row_begin", ctypes.c_int64), ("row_end", ctypes.c_int64), ("lda", ctypes.c_int64),
                ("flags", ctypes.c_int32), ("uniform", ctypes.c_int32), ("assemble_ms", ctypes.c_double)]


class HMatrixInfo(ctypes.Structure):
    _fields_ = [("nblocks_dense", ctypes.c_int32), ("nblocks_lr", ctypes.c_int32), ("depth", ctypes.c_int32),
                ("nclusters", ctypes.c_int32), ("dense_entries", ctypes.c_int64), ("lr_entries", ctypes.c_int64),
                ("build_ms", ctypes.c_double)]


class HluInfo(ctypes.Structure):
    _fields_ = [("max_rank", ctypes.c_int32), ("stored_entries", ctypes.c_int64), ("factor_ms", ctypes.c_double),
                ("nops", ctypes.c_int32), ("algorithm", ctypes.c_int32),
                ("plan_ms", ctypes.c_double)]


class SolveOpts(ctypes.Structure):
    _fields_ = [("method", ctypes.c_int32), ("tol", ctypes.c_double), ("maxiter", ctypes.c_int32),
                ("restart", ctypes.c_int32), ("path", ctypes.c_int32), ("verify", ctypes.c_int32)]


class SolveReport(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int32), ("matvecs", ctypes.c_int32), ("converged", ctypes.c_int32),
                ("relres", ctypes.c_double), ("solve_ms", ctypes.c_double), ("relres_true", ctypes.c_double)]


def lib_path() -> str:
    return _SO


def lib():
    """Load libfde.so (raises if it is missing: no CPU fallback exists)."""
    global _lib
    if _lib is None:
        so = os.environ.get("FDE_LIB_PATH", _SO)   # (dev A/B of compile-time variants)
        if not os.path.exists(so):
            raise RuntimeError(f"libfde.so not built ({so}); run __graft_entry__.build()")
        L = ctypes.CDLL(so)
        vp, i32, i64, dbl = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_double
        L.fde_create.argtypes = [ctypes.POINTER(vp), i32, vp, vp, i32, i32]
        L.fde_create_virtual_rank.argtypes = [ctypes.POINTER(vp), i32, vp, i32, i32]
        L.fde_operator_rows_internal.argtypes = [vp, vp, vp, i64]
        L.fde_shard_matvec.argtypes = [vp, vp, vp, i64, vp, i64, i32]
        L.fde_debug_compact_gather.argtypes = [vp, vp, vp, vp, i64, i32]
        L.fde_debug_comm_selftest.argtypes = [vp, vp, vp, vp, i64, i32]
        L.fde_debug_truncate.argtypes = [vp, vp, vp, i64, i64, i32, i32, dbl, i32, vp, vp, ctypes.POINTER(i32)]
        L.fde_destroy.argtypes = [vp]
        L.fde_destroy.restype = None
        L.fde_last_error.argtypes = [vp]
        L.fde_last_error.restype = ctypes.c_char_p
        L.fde_sync.argtypes = [vp]
        L.fde_nccl_unique_id.argtypes = [vp]
        L.sem_assemble.argtypes = [vp, ctypes.POINTER(Problem), ctypes.POINTER(Mesh), i32, ctypes.POINTER(vp)]
        L.fde_operator_get_info.argtypes = [vp, ctypes.POINTER(OperatorInfo)]
        L.fde_operator_dense_paper.argtypes = [vp, vp, vp, i64]
        L.fde_operator_boundary_columns.argtypes = [vp, vp, vp]
        L.sem_rhs.argtypes = [vp, vp, ctypes.POINTER(Forcing), i32, vp, i64]
        L.stiffness_matvec.argtypes = [vp, vp, vp, vp, i32, i64, i32]
        L.hmatrix_build.argtypes = [vp, vp, i32, dbl, i32, ctypes.POINTER(vp)]
        L.hmatrix_build_partition.argtypes = [vp, vp, i32, dbl, i32, i32, ctypes.POINTER(vp)]
        L.fde_hmatrix_get_info.argtypes = [vp, ctypes.POINTER(HMatrixInfo)]
        L.fde_hmatrix_dense_paper.argtypes = [vp, vp, vp, i64]
        L.hlu_factor.argtypes = [vp, vp, dbl, ctypes.POINTER(vp)]
        L.fde_hlu_get_info.argtypes = [vp, ctypes.POINTER(HluInfo)]
        L.precond_apply.argtypes = [vp, vp, vp, vp, i32, i64]
        L.fde_hlu_dense_internal.argtypes = [vp, vp, vp, i64]
        L.fde_profile.argtypes = [vp, i32]
        L.fde_profile_collect.argtypes = [vp, ctypes.POINTER(ctypes.c_double), i32]
        L.fde_shard_rows.argtypes = [i32, i32, i32, i32, ctypes.POINTER(i64), ctypes.POINTER(i64),
                                     ctypes.POINTER(i64)]
        L.fde_debug_hlu_mode.argtypes = [i32]
        L.fde_debug_pool_bytes.argtypes = [i32, ctypes.POINTER(ctypes.c_ulonglong), ctypes.POINTER(ctypes.c_ulonglong)]
        L.fde_launch_count.argtypes = []
        L.fde_launch_count.restype = ctypes.c_longlong
        L.solve.argtypes = [vp, vp, vp, vp, vp, i32, i64, ctypes.POINTER(SolveOpts), ctypes.POINTER(SolveReport)]
        L.fde_free_operator.argtypes = [vp]
        L.fde_free_operator.restype = None
        L.fde_free_hmatrix.argtypes = [vp]
        L.fde_free_hmatrix.restype = None
        L.fde_free_hlu.argtypes = [vp]
        L.fde_free_hlu.restype = None
        _lib = L
    return _lib


def _check(rc: int, h=None):
    if rc != 0:
        msg = lib().fde_last_error(h).decode() if True else ""
        raise FdeError(rc, msg)


def _ptr(t) -> int:
    """Device pointer of a tensor argument: the C-ABI takes float64 CUDA buffers with
    the stated strides, so anything else is rejected here (a float32 or host
    tensor would otherwise be read as garbage)."""
    import torch
    if t.dtype != torch.float64:
        raise TypeError(f"fde: expected a float64 tensor, got {t.dtype}")
    if not t.is_cuda:
        raise ValueError("fde: expected a CUDA tensor (device buffers cross the C-ABI)")
    if not t.is_contiguous():
        raise ValueError("fde: expected a contiguous tensor")
    return t.data_ptr()


class Handle:
    """fde_create on the current torch CUDA stream (one process per GPU)."""

    def __init__(self, device: int = 0, stream: Optional[int] = None, nccl_id: Optional[bytes] = None,
                 rank: int = 0, world: int = 1, virtual: bool = False):
        """virtual=True: fde_create_virtual_rank (rank `rank` of `world` without a
        communicator; test helper for the sharded path on one GPU)."""
        import torch
        if stream is None:
            stream = torch.cuda.current_stream(device).cuda_stream
        self.h = ctypes.c_void_p()
        if virtual:
            rc = lib().fde_create_virtual_rank(ctypes.byref(self.h), device, ctypes.c_void_p(stream), rank, world)
        else:
            idbuf = ctypes.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
            rc = lib().fde_create(ctypes.byref(self.h), device, ctypes.c_void_p(stream),
                                  ctypes.cast(idbuf, ctypes.c_void_p) if idbuf is not None else None, rank, world)
        if rc != 0:
            raise FdeError(rc, lib().fde_last_error(None).decode())
        self.device, self.rank, self.world = device, rank, world

    def sync(self):
        _check(lib().fde_sync(self.h), self.h)

    def close(self):
        if self.h:
            lib().fde_destroy(self.h)
            self.h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def shard_rows(N: int, P: int, world: int, rank: int):
    """(r0, r1, rows_max) of this rank's row block (internal order), host-only."""
    a, b, c = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    _check(lib().fde_shard_rows(N, P, world, rank, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)))
    return a.value, b.value, c.value


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib().fde_nccl_unique_id(buf), None)
    return buf.raw


class Operator:
    def __init__(self, handle: Handle, ptr: ctypes.c_void_p):
        self.handle, self.ptr = handle, ptr
        inf = OperatorInfo()
        _check(lib().fde_operator_get_info(ptr, ctypes.byref(inf)))   # (does not wait)
        self._info = inf
        self.n = inf.n

    @property
    def info(self):
        """Operator facts; assemble_ms is final once the assembly completed (waits for it)."""
        if self._info.assemble_ms < 0:
            _check(lib().fde_operator_wait(self.ptr))
            _check(lib().fde_operator_get_info(self.ptr, ctypes.byref(self._info)))
        return self._info

    def free(self):
        if self.ptr:
            lib().fde_free_operator(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.free()
        except Exception:   # interpreter shutdown: module globals already cleared
            pass


def sem_assemble(handle: Handle, a, b, alpha, theta, rho, c1, c2, nodes: np.ndarray, P: int,
                 flags: int = OP_DENSE, kind: int = MESH_CUSTOM) -> Operator:
    nodes = np.ascontiguousarray(nodes, dtype=np.float64)
    prob = Problem(a, b, alpha, theta, rho, c1, c2)
    mesh = Mesh(len(nodes) - 1, nodes.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), P, kind)
    out = ctypes.c_void_p()
    _check(lib().sem_assemble(handle.h, ctypes.byref(prob), ctypes.byref(mesh), flags, ctypes.byref(out)), handle.h)
    return Operator(handle, out)


def assemble_problem(handle: Handle, prob, flags: int = OP_DENSE) -> Operator:
    """sem_assemble for an fde_inputs.Problem."""
    return sem_assemble(handle, prob.a, prob.b, prob.alpha, prob.theta, prob.rho, prob.c1, prob.c2,
                        prob.nodes, prob.P, flags)


def _forcing_structs(forcings: Sequence) -> tuple:
    keep = []
    arr = (Forcing * len(forcings))()
    for k, f in enumerate(forcings):
        leg = np.ascontiguousarray(f.leg, dtype=np.float64)
        side = np.array([0 if s == "L" else 1 for s, _, _ in f.terms], dtype=np.int32)
        pw = np.array([p for _, p, _ in f.terms], dtype=np.float64)
        cf = np.array([c for _, _, c in f.terms], dtype=np.float64)
        keep += [leg, side, pw, cf]
        dp = ctypes.POINTER(ctypes.c_double)
        arr[k].nleg = len(leg)
        arr[k].leg = leg.ctypes.data_as(dp) if len(leg) else None
        arr[k].nterm = len(cf)
        arr[k].side = side.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)) if len(cf) else None
        arr[k].power = pw.ctypes.data_as(dp) if len(cf) else None
        arr[k].coef = cf.ctypes.data_as(dp) if len(cf) else None
    return arr, keep


def sem_rhs(handle: Handle, op: Operator, forcings: Sequence):
    import torch
    arr, keep = _forcing_structs(forcings)
    G = torch.empty((len(forcings), op.n), dtype=torch.float64, device=f"cuda:{handle.device}")
    _check(lib().sem_rhs(handle.h, op.ptr, arr, len(forcings), _ptr(G), op.n), handle.h)
    return G


def stiffness_matvec(handle: Handle, op: Operator, x, path: int = PATH_AUTO, out=None):
    import torch
    x = x.reshape(-1, op.n).contiguous()
    y = out if out is not None else torch.empty_like(x)
    _check(lib().stiffness_matvec(handle.h, op.ptr, _ptr(x), _ptr(y), x.shape[0], op.n, path), handle.h)
    return y


def operator_dense_paper(handle: Handle, op: Operator):
    import torch
    A = torch.empty((op.n, op.n), dtype=torch.float64, device=f"cuda:{handle.device}")
    _check(lib().fde_operator_dense_paper(handle.h, op.ptr, _ptr(A), op.n), handle.h)
    return A     # row-major: A[I, J]


def operator_rows_internal(handle: Handle, op: Operator):
    """This rank's dense rows (internal order), shape (row_end - row_begin, n)."""
    import torch
    inf = op.info
    A = torch.empty((max(inf.row_end - inf.row_begin, 0), op.n), dtype=torch.float64, device=f"cuda:{handle.device}")
    _check(lib().fde_operator_rows_internal(handle.h, op.ptr, _ptr(A), op.n), handle.h)
    return A


def shard_matvec(handle: Handle, op: Operator, x, rows_max: int):
    """Local rows of A x (internal order) on this rank's shard: (nrhs, rows_max)."""
    import torch
    x = x.reshape(-1, op.n).contiguous()
    y = torch.zeros((x.shape[0], rows_max), dtype=torch.float64, device=x.device)
    _check(lib().fde_shard_matvec(handle.h, op.ptr, _ptr(x), op.n, _ptr(y), rows_max, x.shape[0]), handle.h)
    return y


def compact_gather(handle: Handle, op: Operator, gathered, nrhs: int):
    """The post-all-gather compaction on a (world, nrhs, rows_max) buffer -> (nrhs, n) paper order."""
    import torch
    g = gathered.contiguous()
    y = torch.empty((nrhs, op.n), dtype=torch.float64, device=g.device)
    _check(lib().fde_debug_compact_gather(handle.h, op.ptr, _ptr(g), _ptr(y), op.n, nrhs), handle.h)
    return y


def comm_selftest(handle: Handle, op: Operator, x):
    """A x through a one-rank NCCL communicator (ncclAllGather + compaction), world-1 handle."""
    import torch
    x = x.contiguous()
    y = torch.empty_like(x)
    _check(lib().fde_debug_comm_selftest(handle.h, op.ptr, _ptr(x), _ptr(y), op.n, x.shape[0]), handle.h)
    return y


def truncate(handle: Handle, U, V, tol: float, kc: int):
    """The H-LU's batched truncation of nb sums U_q V_q^T: U (nb, k, m), V (nb, k, n)
    (rows of the torch tensors = columns of the column-major blocks) -> (Uo, Vo,
    overflow) with Uo (nb, kc, m), Vo (nb, kc, n)."""
    import torch
    U = U.contiguous()
    V = V.contiguous()
    nb, k, m = U.shape
    n = V.shape[2]
    Uo = torch.empty((nb, kc, m), dtype=torch.float64, device=U.device)
    Vo = torch.empty((nb, kc, n), dtype=torch.float64, device=U.device)
    ov = ctypes.c_int32(0)
    _check(lib().fde_debug_truncate(handle.h, _ptr(U), _ptr(V), m, n, k, nb, tol, kc, _ptr(Uo), _ptr(Vo),
                                    ctypes.byref(ov)), handle.h)
    return Uo, Vo, bool(ov.value)


def operator_boundary_columns(handle: Handle, op: Operator):
    import torch
    B = torch.empty((2, op.n), dtype=torch.float64, device=f"cuda:{handle.device}")
    _check(lib().fde_operator_boundary_columns(handle.h, op.ptr, _ptr(B)), handle.h)
    return B


class HMatrix:
    def __init__(self, handle, ptr, n, op=None):
        # the library's H-matrix points at its operator (fde.h lifetime rule):
        # keep the Python object alive as long as this one
        self.handle, self.ptr, self.n, self._op = handle, ptr, n, op
        inf = HMatrixInfo()
        _check(lib().fde_hmatrix_get_info(ptr, ctypes.byref(inf)))   # (does not wait)
        self._info = inf

    @property
    def info(self):
        """H-matrix facts; build_ms is final once the build completed (waits for it)."""
        if self._info.build_ms < 0:
            _check(lib().fde_hmatrix_wait(self.ptr))
            _check(lib().fde_hmatrix_get_info(self.ptr, ctypes.byref(self._info)))
        return self._info

    def free(self):
        if self.ptr:
            lib().fde_free_hmatrix(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.free()
        except Exception:   # interpreter shutdown: module globals already cleared
            pass


def hmatrix_build(handle: Handle, op: Operator, R: int, lam: float = 1.0, n_min: int = 16,
                  partition: int = PARTITION_INTERLEAVED) -> HMatrix:
    """partition: PARTITION_INTERLEAVED (default, reading A9) or PARTITION_PAPER
    (separate modal / nodal trees)."""
    out = ctypes.c_void_p()
    if partition == PARTITION_INTERLEAVED:
        _check(lib().hmatrix_build(handle.h, op.ptr, R, lam, n_min, ctypes.byref(out)), handle.h)
    else:
        _check(lib().hmatrix_build_partition(handle.h, op.ptr, R, lam, n_min, partition, ctypes.byref(out)), handle.h)
    return HMatrix(handle, out, op.n, op)


def hmatrix_dense_paper(handle: Handle, hm: HMatrix):
    import torch
    A = torch.empty((hm.n, hm.n), dtype=torch.float64, device=f"cuda:{handle.device}")
    _check(lib().fde_hmatrix_dense_paper(handle.h, hm.ptr, _ptr(A), hm.n), handle.h)
    return A.t()   # column-major buffer -> [I, J]


class HLU:
    def __init__(self, handle, ptr, n, hm=None):
        # keeps its H-matrix (and through it the operator) alive: fde.h lifetime rule
        self.handle, self.ptr, self.n, self._hm = handle, ptr, n, hm
        inf = HluInfo()
        _check(lib().fde_hlu_get_info(ptr, ctypes.byref(inf)))
        self.info = inf

    def free(self):
        if self.ptr:
            lib().fde_free_hlu(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.free()
        except Exception:   # interpreter shutdown: module globals already cleared
            pass


def hlu_factor(handle: Handle, hm: HMatrix, tol: float = 1e-3) -> HLU:
    out = ctypes.c_void_p()
    _check(lib().hlu_factor(handle.h, hm.ptr, tol, ctypes.byref(out)), handle.h)
    return HLU(handle, out, hm.n, hm)


def hlu_dense_internal(handle: Handle, lu: HLU):
    import torch
    F = torch.zeros((lu.n, lu.n), dtype=torch.float64, device=f"cuda:{handle.device}")
    _check(lib().fde_hlu_dense_internal(handle.h, lu.ptr, _ptr(F), lu.n), handle.h)
    return F.t()   # column-major buffer -> [I, J]


def internal_to_paper_index(N: int, P: int):
    """paper index of every internal (element-interleaved) dof (fde.h convention)."""
    import numpy as np
    r = np.arange(N * P - 1)
    e, q = r // P, r % P
    return np.where(q < P - 1, e * (P - 1) + q, N * (P - 1) + e)


def precond_apply(handle: Handle, lu: HLU, r, out=None):
    import torch
    r = r.reshape(-1, lu.n).contiguous()
    z = out if out is not None else torch.empty_like(r)
    _check(lib().precond_apply(handle.h, lu.ptr, _ptr(r), _ptr(z), r.shape[0], lu.n), handle.h)
    return z


def solve(handle: Handle, op: Operator, lu: Optional[HLU], G, method: int = GMRES, tol: float = 1e-12,
          maxiter: int = 500, restart: int = 50, path: int = PATH_AUTO, out=None, verify: bool = True):
    """X = solve(A~^{-1} A X = A~^{-1} G); returns (X, report).  verify (GMRES):
    confirm convergence on the recomputed preconditioned residual (report.relres_true)."""
    import torch
    G = G.reshape(-1, op.n).contiguous()
    X = out if out is not None else torch.empty_like(G)
    o = SolveOpts(method, tol, maxiter, restart, path, 1 if verify else 0)
    rep = SolveReport()
    _check(lib().solve(handle.h, op.ptr, lu.ptr if lu is not None else None, _ptr(G), _ptr(X), G.shape[0], op.n,
                       ctypes.byref(o), ctypes.byref(rep)), handle.h)
    return X, rep


def set_hlu_mode(mode: int) -> None:
    """0: leaf-ordered batched H-LU when the partition allows it (default), 1: recursive only."""
    _check(lib().fde_debug_hlu_mode(int(mode)))


def pool_bytes(device: int = 0):
    """(reserved, used) bytes of the device's default memory pool (diagnostics)."""
    r, u = ctypes.c_ulonglong(), ctypes.c_ulonglong()
    _check(lib().fde_debug_pool_bytes(int(device), ctypes.byref(r), ctypes.byref(u)))
    return r.value, u.value
