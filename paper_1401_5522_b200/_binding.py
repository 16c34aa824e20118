"""ctypes binding of include/hlq.h (marshalling only: every step of the path runs in libhlq.so).

Device buffers are torch CUDA float64 tensors used purely as memory: an N x N column-major matrix
is a contiguous tensor whose storage holds A in LAPACK order (see `to_colmajor`).  Streams are torch
CUDA streams (the current stream by default).
"""
from __future__ import annotations

import ctypes as C
import math
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
lib_path = os.path.join(_HERE, "libhlq.so")

CRIT_MAX, CRIT_SUM, CRIT_MUMPS, CRIT_RANDOM = 0, 1, 2, 3
DEC_LU, DEC_QR = 0, 1
LU_A1, LU_A2 = 0, 1  # hlq_options.lu_variant (NEXT f4)
PIVOT_TILE, PIVOT_DOMAIN = 0, 1  # hlq_options.pivot_scope (NEXT f1)
TREE_GREEDY, TREE_HQR = 0, 1  # hlq_options.tree (HQR: TS groups of ts_group tiles)
FLAG_ZERO_PIVOT, FLAG_NEAR_TIE, FLAG_FORCED, FLAG_HINTED, FLAG_NONFINITE = 1, 2, 4, 8, 16


class HlqError(RuntimeError):
    pass


class HlqOptions(C.Structure):
    _fields_ = [("struct_size", C.c_int32), ("lda", C.c_int64), ("ib", C.c_int32),
                ("tree_domains", C.c_int32), ("tree", C.c_int32), ("mumps_reading", C.c_int32),
                ("forced", C.c_void_p), ("ref_dec", C.c_void_p), ("ref_margin", C.c_void_p),
                ("tie_rel_tol", C.c_double), ("track_growth", C.c_int32), ("blocking", C.c_int32),
                ("stream", C.c_void_p), ("profile", C.c_int32), ("invnorm_estimate", C.c_int32),
                ("lu_variant", C.c_int32), ("pivot_scope", C.c_int32), ("ts_group", C.c_int32)]


class HlqInfo(C.Structure):
    _fields_ = [("N", C.c_int64), ("nb", C.c_int32), ("n", C.c_int32), ("ib", C.c_int32),
                ("D", C.c_int32), ("qr_steps", C.c_int32), ("near_ties", C.c_int32),
                ("hinted", C.c_int32), ("status", C.c_int32), ("growth", C.c_double),
                ("fake_flops", C.c_double), ("true_flops", C.c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


def _load():
    if not os.path.exists(lib_path):
        raise HlqError(f"libhlq.so not built at {lib_path}: run `python -c 'import __graft_entry__ as g;"
                       f" g.build()'` (no CPU fallback exists)")
    L = C.CDLL(lib_path)
    P, I32, I64, D, U64 = C.c_void_p, C.c_int32, C.c_int64, C.c_double, C.c_uint64
    sig = {
        "hlq_abi": ([P, P, P], I32),
        "hlq_default_options": ([P], I32),
        "hlq_factor": ([P, I64, I32, I32, D, P], I32),
        "hlq_factor_ex": ([P, I64, I32, I32, D, P, P], I32),
        "hlq_solve": ([P, P, P], I32),
        "hlq_gesv_host": ([P, P, P, I64, I32, I32, D, P, P], I32),
        "hlq_get_info": ([P, P], I32),
        "hlq_get_decisions": ([P, P], I32),
        "hlq_get_margins": ([P, P], I32),
        "hlq_get_step_flags": ([P, P], I32),
        "hlq_get_step_log": ([P, P], I32),
        "hlq_get_step_times": ([P, P], I32),
        "hlq_get_growth": ([P, P], I32),
        "hlq_get_pivots": ([P, P], I32),
        "hlq_get_T": ([P, I32, I32, I32, P], I32),
        "hlq_free": ([P], None),
        "hlq_status_string": ([I32], C.c_char_p),
        "hlq_generate_uniform": ([P, I64, I64, I64, U64, U64, I64, P], I32),
        "hlq_residual": ([P, I64, I64, P, P, P, P], I32),
        "hlq_get_profile": ([P, P, P, P], I32),
        "hlq_launch_count": ([], I64),
        "hlq_test_schur": ([P, I64, I64, I64, I32, I32, P], I32),
        "hlq_nccl_unique_id": ([P], I32),
        "hlq_grid_create_nccl": ([P, I32, I32, I32, I32, P], I32),
        "hlq_grid_create_local": ([I32, I32, P], I32),
        "hlq_grid_create_host": ([P, I32, I32, I32, I32, P], I32),
        "hlq_grid_free": ([P], None),
        "hlq_grid_info": ([P, P, P, P, P], I32),
        "hlq_grid_local_shape": ([I64, I32, I32, I32, I32, I32, P, P], I32),
        "hlq_dist_plan": ([I32, I32, I32, I32, I32, P, I32], I32),
        "hlq_dist_counts": ([I64, I32, I32, I32, I32, I32, I32, I32, P], I32),
        "hlq_factor_dist": ([P, P, P, I64, I32, I32, D, P, P], I32),
        "hlq_generate_uniform_cyclic": ([P, P, P, I64, I32, U64, P], I32),
        "hlq_residual_dist": ([P, P, P, I64, I32, P, P, P, P], I32),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    so, si, ver = C.c_int32(), C.c_int32(), C.c_int32()
    L.hlq_abi(C.byref(so), C.byref(si), C.byref(ver))
    if so.value != C.sizeof(HlqOptions) or si.value != C.sizeof(HlqInfo):
        raise HlqError(f"ABI mismatch: C sizeof(options/info) = {so.value}/{si.value}, "
                       f"binding {C.sizeof(HlqOptions)}/{C.sizeof(HlqInfo)}")
    return L


lib = _load()


def _check(rc, what):
    if rc < 0:
        raise HlqError(f"{what} failed: {rc} ({lib.hlq_status_string(rc).decode()})")
    return rc


def hlq_abi():
    so, si, ver = C.c_int32(), C.c_int32(), C.c_int32()
    lib.hlq_abi(C.byref(so), C.byref(si), C.byref(ver))
    return so.value, si.value, ver.value


def hlq_default_options() -> HlqOptions:
    o = HlqOptions()
    lib.hlq_default_options(C.byref(o))
    return o


def _stream_ptr(stream):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _dptr(t):
    return C.c_void_p(t.data_ptr())


# ------------------------------------------------------------------- layout helpers (plumbing)
def to_colmajor(A_host: np.ndarray, device="cuda"):
    """numpy (N x N) -> torch CUDA tensor whose storage is A in column-major (LAPACK) order."""
    import torch
    AT = np.ascontiguousarray(np.asarray(A_host, dtype=np.float64).T)
    return torch.from_numpy(AT).to(device)


def from_colmajor(t) -> np.ndarray:
    """inverse of to_colmajor (device tensor -> numpy N x N)."""
    return t.detach().cpu().numpy().T


class Factors:
    """Owns an hlq_factors_t handle (the factorization borrows the device matrix `A`)."""

    def __init__(self, handle, A, status, keep=()):
        self.handle = C.c_void_p(handle)
        self.A = A
        self.status = status
        self._keep = keep

    def __del__(self):
        self.free()

    def free(self):
        if getattr(self, "handle", None) and self.handle.value:
            lib.hlq_free(self.handle)
            self.handle = C.c_void_p(None)

    def info(self) -> dict:
        inf = HlqInfo()
        _check(lib.hlq_get_info(self.handle, C.byref(inf)), "hlq_get_info")
        return inf.as_dict()

    @property
    def n(self):
        return self.info()["n"]

    def decisions(self) -> np.ndarray:
        d = np.zeros(self.n, dtype=np.uint8)
        _check(lib.hlq_get_decisions(self.handle, d.ctypes.data_as(C.c_void_p)), "decisions")
        return d

    def margins(self) -> np.ndarray:
        m = np.zeros(self.n, dtype=np.float64)
        _check(lib.hlq_get_margins(self.handle, m.ctypes.data_as(C.c_void_p)), "margins")
        return m

    def step_flags(self) -> np.ndarray:
        f = np.zeros(self.n, dtype=np.int32)
        _check(lib.hlq_get_step_flags(self.handle, f.ctypes.data_as(C.c_void_p)), "flags")
        return f

    def step_log(self) -> np.ndarray:
        """n x 2: the two sides of each step's binding criterion inequality (NaN: no criterion)."""
        v = np.zeros(2 * self.n, dtype=np.float64)
        _check(lib.hlq_get_step_log(self.handle, v.ctypes.data_as(C.c_void_p)), "step_log")
        return v.reshape(-1, 2)

    def step_times(self) -> np.ndarray:
        """per-step device ms (profiled handles only)."""
        v = np.zeros(self.n, dtype=np.float64)
        _check(lib.hlq_get_step_times(self.handle, v.ctypes.data_as(C.c_void_p)), "step_times")
        return v

    def growth(self) -> float:
        g = C.c_double()
        _check(lib.hlq_get_growth(self.handle, C.byref(g)), "growth")
        return g.value

    def pivots(self) -> np.ndarray:
        inf = self.info()
        p = np.zeros(inf["n"] * inf["nb"], dtype=np.int32)
        _check(lib.hlq_get_pivots(self.handle, p.ctypes.data_as(C.c_void_p)), "pivots")
        return p.reshape(inf["n"], inf["nb"])

    def T(self, i, k, kind=0) -> np.ndarray:
        inf = self.info()
        t = np.zeros(inf["ib"] * inf["nb"], dtype=np.float64)
        _check(lib.hlq_get_T(self.handle, i, k, kind, t.ctypes.data_as(C.c_void_p)), "T")
        return t.reshape(inf["nb"], inf["ib"]).T

    PROF_CLASSES = ("criterion", "getrf", "lu_trsm", "lu_update", "qr_geqrt", "qr_unmqr",
                    "qr_tt", "growth", "solve", "other")

    def profile(self) -> dict:
        ms = np.zeros(10)
        fl = np.zeros(10)
        ln = np.zeros(10, dtype=np.int64)
        rc = lib.hlq_get_profile(self.handle, ms.ctypes.data_as(C.c_void_p),
                                 fl.ctypes.data_as(C.c_void_p), ln.ctypes.data_as(C.c_void_p))
        _check(rc, "hlq_get_profile")
        return {c: {"ms": float(ms[i]), "flops": float(fl[i]), "launches": int(ln[i])}
                for i, c in enumerate(self.PROF_CLASSES)}

    def solve(self, b, x=None):
        import torch
        if x is None:
            x = torch.empty_like(b)
        hlq_solve(self, b, x)
        return x


def _check_device_matrix(A, rows: int, cols: int, ld: int, what: str):
    """A must be a contiguous float64 CUDA tensor holding at least ld*(cols-1)+rows elements."""
    import torch
    if not isinstance(A, torch.Tensor):
        raise HlqError(f"{what}: expected a torch tensor, got {type(A).__name__}")
    if A.dtype != torch.float64 or not A.is_cuda or not A.is_contiguous():
        raise HlqError(f"{what}: needs a contiguous float64 CUDA tensor "
                       f"(got {A.dtype}, device {A.device}, contiguous={A.is_contiguous()})")
    need = ld * (cols - 1) + rows if rows > 0 and cols > 0 else 0
    if A.numel() < need:
        raise HlqError(f"{what}: {A.numel()} elements < ld*(N-1)+N = {need}")


def _step_vectors(opt: HlqOptions, n: int, forced, ref_dec, ref_margin, keep: list):
    """Marshal the per-step host vectors (n entries each) into opt."""
    if forced is not None:
        fa = np.ascontiguousarray(forced, dtype=np.uint8)
        if fa.shape != (n,):
            raise HlqError(f"forced has shape {fa.shape}, needs ({n},) = ceil(N/nb)")
        keep.append(fa)
        opt.forced = fa.ctypes.data
    if (ref_dec is None) != (ref_margin is None):
        raise HlqError("ref_dec and ref_margin must be given together")
    if ref_dec is not None:
        ra = np.ascontiguousarray(ref_dec, dtype=np.uint8)
        rm = np.ascontiguousarray(ref_margin, dtype=np.float64)
        if ra.shape != (n,) or rm.shape != (n,):
            raise HlqError(f"ref_dec / ref_margin have shapes {ra.shape} / {rm.shape}, need ({n},)")
        keep += [ra, rm]
        opt.ref_dec = ra.ctypes.data
        opt.ref_margin = rm.ctypes.data


def hlq_factor_ex(A, N: int, nb: int, criterion: int = CRIT_MAX, alpha: float = 1.0,
                  opt: HlqOptions | None = None, *, forced=None, ref_dec=None, ref_margin=None,
                  stream=None, **fields) -> Factors:
    """Factor the device matrix A (torch float64 CUDA tensor, column-major storage) in place."""
    if opt is None:
        opt = hlq_default_options()
    for k, v in fields.items():
        setattr(opt, k, v)
    if N >= 1 and nb >= 1:
        _check_device_matrix(A, N, N, opt.lda if opt.lda else N, "hlq_factor_ex: A")
    keep = []
    n = -(-N // min(nb, N)) if N >= 1 and nb >= 1 else 0
    _step_vectors(opt, n, forced, ref_dec, ref_margin, keep)
    opt.stream = _stream_ptr(stream).value
    h = C.c_void_p()
    rc = lib.hlq_factor_ex(_dptr(A), N, nb, criterion, float(alpha), C.byref(opt), C.byref(h))
    if rc < 0:
        if h.value:
            lib.hlq_free(h)
        _check(rc, "hlq_factor_ex")
    return Factors(h.value, A, rc, tuple(keep))


def hlq_factor(A, N: int, nb: int, criterion: int = CRIT_MAX, alpha: float = 1.0) -> Factors:
    return hlq_factor_ex(A, N, nb, criterion, alpha)


def hlq_test_schur(A, N: int, lda: int, k0: int, K: int, use_tma: bool, stream=None) -> int:
    """One LU Schur update on the device matrix A (test hook; 1 = the TMA kernel ran)."""
    return _check(lib.hlq_test_schur(_dptr(A), N, lda, k0, K, int(use_tma), _stream_ptr(stream)),
                  "hlq_test_schur")


def hlq_launch_count() -> int:
    return int(lib.hlq_launch_count())


def hlq_solve(f: Factors, b, x):
    N = f.info()["N"]
    _check_device_matrix(b, N, 1, N, "hlq_solve: b")
    _check_device_matrix(x, N, 1, N, "hlq_solve: x")
    return _check(lib.hlq_solve(f.handle, _dptr(b), _dptr(x)), "hlq_solve")


def hlq_gesv_host(A_host: np.ndarray, b_host: np.ndarray, x_host: np.ndarray, N: int, nb: int,
                  criterion: int = CRIT_MAX, alpha: float = 1.0, opt: HlqOptions | None = None,
                  stream=None):
    """Host buffers (A column-major, i.e. a Fortran-ordered numpy array or its raw storage)."""
    if opt is None:
        opt = hlq_default_options()
    opt.stream = _stream_ptr(stream).value
    info = HlqInfo()
    rc = lib.hlq_gesv_host(C.c_void_p(A_host.ctypes.data), C.c_void_p(b_host.ctypes.data),
                           C.c_void_p(x_host.ctypes.data), N, nb, criterion, float(alpha),
                           C.byref(opt), C.byref(info))
    _check(rc, "hlq_gesv_host")
    return rc, info.as_dict()


def hlq_generate_uniform(dst, rows, cols, ld, seed, idx0, idx_ld, stream=None):
    _check(lib.hlq_generate_uniform(_dptr(dst), rows, cols, ld, seed, idx0, idx_ld,
                                    _stream_ptr(stream)), "hlq_generate_uniform")


def hlq_residual(A, N, lda, x, b, stream=None):
    out = np.zeros(3)
    _check(lib.hlq_residual(_dptr(A), N, lda, _dptr(x), _dptr(b), out.ctypes.data_as(C.c_void_p),
                            _stream_ptr(stream)), "hlq_residual")
    r, an, xn = out
    return {"resid_inf": r, "A_inf": an, "x_inf": xn,
            "hpl3": r / (an * xn * 2.0 ** -53 * N) if an * xn > 0 else math.inf}


# ------------------------------------------------------------------ 2D block-cyclic (row e)
def local_shape(N: int, nb: int, P: int, Q: int, p: int, q: int):
    """(mloc, nloc) of rank (p, q) (host-only)."""
    m, n = C.c_int64(), C.c_int64()
    _check(lib.hlq_grid_local_shape(N, nb, P, Q, p, q, C.byref(m), C.byref(n)), "local_shape")
    return m.value, n.value


def cyclic_rows(N: int, nb: int, P: int, p: int) -> np.ndarray:
    """global row (or column) indices held by process row p, in local order (plumbing)."""
    n = -(-N // nb)
    parts = [np.arange(i * nb, min((i + 1) * nb, N)) for i in range(p, n, P)]
    return np.concatenate(parts) if parts else np.zeros(0, dtype=np.int64)


def scatter_block_cyclic(A: np.ndarray, nb: int, P: int, Q: int, p: int, q: int) -> np.ndarray:
    N = A.shape[0]
    return A[np.ix_(cyclic_rows(N, nb, P, p), cyclic_rows(N, nb, Q, q))]


def gather_block_cyclic(locs: dict, N: int, nb: int, P: int, Q: int) -> np.ndarray:
    """locs[(p, q)] = local numpy array -> global N x N."""
    A = np.zeros((N, N))
    for (p, q), L in locs.items():
        if L.size == 0:
            continue
        A[np.ix_(cyclic_rows(N, nb, P, p), cyclic_rows(N, nb, Q, q))] = L
    return A


def dist_plan(n: int, P: int, D: int, p: int, k: int) -> dict:
    """parsed hlq_dist_plan (host-only)."""
    ln = lib.hlq_dist_plan(n, P, D, p, k, None, 0)
    _check(ln, "hlq_dist_plan")
    buf = np.zeros(ln, dtype=np.int32)
    lib.hlq_dist_plan(n, P, D, p, k, buf.ctypes.data_as(C.c_void_p), ln)
    v = buf.tolist()
    out = {"li0": v[0], "ms": v[1], "diag": v[2]}
    c = v[3]
    pos = 4
    out["heads"] = [(v[pos + 2 * t], v[pos + 2 * t + 1]) for t in range(c)]
    pos += 2 * c

    def levels():
        nonlocal pos
        nl = v[pos]
        pos += 1
        lv = []
        for _ in range(nl):
            cnt = v[pos]
            pos += 1
            lv.append([(v[pos + 2 * j], v[pos + 2 * j + 1]) for j in range(cnt)])
            pos += 2 * cnt
        return lv

    out["intra"] = levels()
    out["inter"] = levels()
    return out


def dist_counts(N: int, nb: int, P: int, Q: int, D: int, p: int, q: int, k: int):
    """(stats record, head tiles, panel package, head rows) element counts of step k (host-only)."""
    out = np.zeros(4, dtype=np.int64)
    _check(lib.hlq_dist_counts(N, nb, P, Q, D, p, q, k, out.ctypes.data_as(C.c_void_p)),
           "hlq_dist_counts")
    return tuple(int(v) for v in out)


class Grid:
    """Owns an hlq_grid_t: NCCL (one process per GPU) or emulated (all ranks in this process)."""

    def __init__(self, handle):
        self.handle = C.c_void_p(handle)
        P, Q, nl, r0 = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
        _check(lib.hlq_grid_info(self.handle, C.byref(P), C.byref(Q), C.byref(nl), C.byref(r0)),
               "hlq_grid_info")
        self.P, self.Q, self.nlocal, self.rank0 = P.value, Q.value, nl.value, r0.value

    def ranks(self):
        """(p, q) of the ranks hosted here, in the order hlq_factor_dist expects."""
        return [divmod(self.rank0 + t, self.Q) for t in range(self.nlocal)]

    def __del__(self):
        self.free()

    def free(self):
        if getattr(self, "handle", None) and self.handle.value:
            lib.hlq_grid_free(self.handle)
            self.handle = C.c_void_p(None)


HC_ALLGATHER = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_int64)
HC_BROADCAST = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int32, C.c_void_p, C.c_int64, C.c_int32)
HC_ALLREDUCE = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int32, C.c_void_p, C.c_int64, C.c_int32)
COMM_WORLD, COMM_ROW, COMM_COL, COMM_COL_PANEL = 0, 1, 2, 3


class HostComm(C.Structure):
    _fields_ = [("struct_size", C.c_int32), ("ctx", C.c_void_p), ("allgather", HC_ALLGATHER),
                ("broadcast", HC_BROADCAST), ("allreduce", HC_ALLREDUCE)]


def grid_host(nranks: int, rank: int, P: int, Q: int, allgather, broadcast, allreduce) -> Grid:
    """Host-staged grid (hlq_grid_create_host): the collectives are the caller's Python functions on
    numpy views of the library's pinned host buffers:
      allgather(comm, send: ndarray[count], recv: ndarray[size*count]),
      broadcast(comm, buf: ndarray[count], root), allreduce(comm, buf: ndarray[count], op)."""
    def ag(ctx, comm, send, recv, count):
        try:
            s = np.ctypeslib.as_array(C.cast(send, C.POINTER(C.c_double)), shape=(count,))
            size = Q if comm == COMM_ROW else (P * Q if comm == COMM_WORLD else P)
            r = np.ctypeslib.as_array(C.cast(recv, C.POINTER(C.c_double)), shape=(size * count,))
            allgather(comm, s, r)
            return 0
        except Exception as e:  # noqa: BLE001  (reported to the library as a failed collective)
            print("hlq host allgather:", repr(e))
            return 1

    def bc(ctx, comm, buf, count, root):
        try:
            v = np.ctypeslib.as_array(C.cast(buf, C.POINTER(C.c_double)), shape=(count,))
            broadcast(comm, v, root)
            return 0
        except Exception as e:  # noqa: BLE001
            print("hlq host broadcast:", repr(e))
            return 1

    def ar(ctx, comm, buf, count, op):
        try:
            v = np.ctypeslib.as_array(C.cast(buf, C.POINTER(C.c_double)), shape=(count,))
            allreduce(comm, v, op)
            return 0
        except Exception as e:  # noqa: BLE001
            print("hlq host allreduce:", repr(e))
            return 1

    ops = HostComm(C.sizeof(HostComm), None, HC_ALLGATHER(ag), HC_BROADCAST(bc), HC_ALLREDUCE(ar))
    h = C.c_void_p()
    _check(lib.hlq_grid_create_host(C.byref(ops), nranks, rank, P, Q, C.byref(h)),
           "hlq_grid_create_host")
    g = Grid(h.value)
    g._ops = ops  # the callbacks must outlive the grid
    return g


def grid_local(P: int, Q: int) -> Grid:
    h = C.c_void_p()
    _check(lib.hlq_grid_create_local(P, Q, C.byref(h)), "hlq_grid_create_local")
    return Grid(h.value)


def nccl_unique_id() -> bytes:
    buf = (C.c_char * 128)()
    _check(lib.hlq_nccl_unique_id(buf), "hlq_nccl_unique_id")
    return bytes(buf)


def grid_nccl(uid: bytes, nranks: int, rank: int, P: int, Q: int) -> Grid:
    buf = (C.c_char * 128).from_buffer_copy(uid)
    h = C.c_void_p()
    _check(lib.hlq_grid_create_nccl(buf, nranks, rank, P, Q, C.byref(h)), "hlq_grid_create_nccl")
    return Grid(h.value)


def hlq_factor_dist(grid: Grid, A_locals, N: int, nb: int, criterion: int = CRIT_MAX,
                    alpha: float = 1.0, opt: HlqOptions | None = None, *, lld=None, forced=None,
                    ref_dec=None, ref_margin=None, stream=None, **fields) -> Factors:
    """Factor the 2D block-cyclic matrix whose local arrays (torch float64 CUDA tensors with
    column-major storage, one per rank hosted here) are A_locals, in place."""
    if opt is None:
        opt = hlq_default_options()
        opt.tree_domains = 0
    for k, v in fields.items():
        setattr(opt, k, v)
    keep = []
    n = -(-N // min(nb, N)) if N >= 1 and nb >= 1 else 0
    _step_vectors(opt, n, forced, ref_dec, ref_margin, keep)
    opt.stream = _stream_ptr(stream).value
    ptrs = (C.c_void_p * len(A_locals))(*[t.data_ptr() if t.numel() else None for t in A_locals])
    llds = (C.c_int64 * len(A_locals))(*([0] * len(A_locals) if lld is None else lld))
    h = C.c_void_p()
    rc = lib.hlq_factor_dist(grid.handle, ptrs, llds, N, nb, criterion, float(alpha), C.byref(opt),
                             C.byref(h))
    if rc < 0:
        if h.value:
            lib.hlq_free(h)
        _check(rc, "hlq_factor_dist")
    return Factors(h.value, list(A_locals), rc, tuple(keep) + (grid,))


def _ptr_array(ts):
    return (C.c_void_p * len(ts))(*[t.data_ptr() if t.numel() else None for t in ts])


def hlq_generate_uniform_cyclic(grid: Grid, A_locals, N: int, nb: int, seed: int, stream=None):
    _check(lib.hlq_generate_uniform_cyclic(grid.handle, _ptr_array(A_locals), None, N, nb, seed,
                                           _stream_ptr(stream)), "hlq_generate_uniform_cyclic")


def hlq_residual_dist(grid: Grid, A_locals, N: int, nb: int, x, b, stream=None):
    out = np.zeros(3)
    _check(lib.hlq_residual_dist(grid.handle, _ptr_array(A_locals), None, N, nb, _dptr(x),
                                 _dptr(b), out.ctypes.data_as(C.c_void_p), _stream_ptr(stream)),
           "hlq_residual_dist")
    r, an, xn = out
    return {"resid_inf": r, "A_inf": an, "x_inf": xn,
            "hpl3": r / (an * xn * 2.0 ** -53 * N) if an * xn > 0 else math.inf}
