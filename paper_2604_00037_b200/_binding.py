"""ctypes binding of libaci.so (include/aci.h). Argument marshalling only: every step of the
ACI path runs in the CUDA kernels behind the C-ABI. There is no CPU fallback — if the library
or a sm_100 device is missing, calls raise.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# ACI_LIB overrides the library path (A/B measurements of two builds)
LIB_PATH = os.environ.get("ACI_LIB", os.path.join(_HERE, "libaci.so"))

ACI_OK, ACI_NOT_CONVERGED = 0, 1
ERRORS = {-1: "ACI_ERR_INVALID", -2: "ACI_ERR_SHAPE", -3: "ACI_ERR_NONFINITE", -4: "ACI_ERR_OOM",
          -5: "ACI_ERR_CUDA", -6: "ACI_ERR_UNSUPPORTED"}
TOL_RELATIVE, TOL_ABSOLUTE = 0, 1
PIVOT_FULL, PIVOT_ROOK = 0, 1
_PIVOTING = {"full": PIVOT_FULL, "rook": PIVOT_ROOK}
MAX_INPUTS, MAX_TERMS, MAX_EXPO = 4, 8, 4

# every symbol include/aci.h declares (tests check the library exports all of them)
EXPORTS = ["tt_create", "tt_create_z", "tt_create_device", "tt_create_device_z", "tt_is_complex", "tt_destroy",
           "tt_shape", "tt_get_cores", "tt_device_cores", "tt_evaluate", "tt_evaluate_device", "aci_elementwise",
           "aci_elementwise_ex", "aci_elementwise_batch", "aci_workspace_query", "aci_limits", "aci_prrlu", "aci_last_error", "aci_version"]


class AciError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code


class aci_op(C.Structure):
    _fields_ = [("n_terms", C.c_int), ("coef", C.POINTER(C.c_double)), ("expo", C.POINTER(C.c_int))]


class aci_report(C.Structure):
    _fields_ = [("error_estimate", C.c_double), ("scale", C.c_double), ("iterations", C.c_int),
                ("converged", C.c_int), ("max_rank", C.c_int), ("n_updates", C.c_int),
                ("pivot_steps", C.c_int64), ("flops_contraction", C.c_double), ("flops_prrlu", C.c_double),
                ("flops_trsm", C.c_double), ("flops_init", C.c_double), ("ms", C.c_float),
                ("n_launches", C.c_int64), ("graph_iterations", C.c_int), ("ms_graph_setup", C.c_float)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class aci_pivot_log(C.Structure):
    _fields_ = [("capacity_updates", C.c_int), ("capacity_pivots", C.c_int), ("info", C.POINTER(C.c_int)),
                ("eps_scale", C.POINTER(C.c_double)), ("rows", C.POINTER(C.c_int)), ("cols", C.POINTER(C.c_int)),
                ("n_written", C.c_int), ("canon_n", C.POINTER(C.c_int)), ("canon_cols", C.POINTER(C.c_int))]


PROF_CLASSES = ["canon", "gemm_ab", "gemm_pi", "prrlu", "update", "conv", "trsm"]


class aci_profile(C.Structure):
    _fields_ = [("ms", C.c_double * 7), ("launches", C.c_int64 * 7)]

    def as_dict(self):
        return {k: {"ms": self.ms[i], "launches": int(self.launches[i])} for i, k in enumerate(PROF_CLASSES)}


class aci_options(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("y_init", C.c_void_p), ("tol_mode", C.c_int),
                ("log", C.POINTER(aci_pivot_log)), ("stream", C.c_void_p), ("workspace", C.c_void_p),
                ("workspace_bytes", C.c_size_t), ("I_sets", C.POINTER(C.POINTER(C.c_uint8))),
                ("J_sets", C.POINTER(C.POINTER(C.c_uint8))), ("profile", C.POINTER(aci_profile)),
                ("iter_ms", C.POINTER(C.c_float)), ("concurrent", C.c_int), ("pivoting", C.c_int)]


_lib = None


def load(path: str = LIB_PATH):
    """Load libaci.so (raises if it is missing: the product path has no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = C.CDLL(path)
    vp, ip, dp = C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_double)
    lib.tt_create.argtypes = [C.c_int, ip, ip, C.POINTER(dp), C.POINTER(vp)]
    lib.tt_create_z.argtypes = [C.c_int, ip, ip, C.POINTER(dp), C.POINTER(vp)]
    lib.tt_create_device.argtypes = [C.c_int, ip, ip, C.c_void_p, C.c_void_p, C.POINTER(vp)]
    lib.tt_create_device_z.argtypes = [C.c_int, ip, ip, C.c_void_p, C.c_void_p, C.POINTER(vp)]
    lib.tt_is_complex.argtypes = [vp]
    lib.tt_destroy.argtypes = [vp]
    lib.tt_shape.argtypes = [vp, ip, ip, ip]
    lib.tt_get_cores.argtypes = [vp, C.POINTER(dp)]
    lib.tt_device_cores.argtypes = [vp]
    lib.tt_device_cores.restype = C.c_void_p
    lib.tt_evaluate.argtypes = [vp, C.c_int64, C.c_void_p, dp]
    lib.tt_evaluate_device.argtypes = [vp, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]
    lib.aci_elementwise.argtypes = [aci_op, C.POINTER(vp), C.c_int, C.c_double, C.c_int, C.c_int, C.POINTER(vp),
                                    C.POINTER(aci_report)]
    lib.aci_elementwise_ex.argtypes = [aci_op, C.POINTER(vp), C.c_int, C.c_double, C.c_int, C.c_int,
                                       C.POINTER(vp), C.POINTER(aci_report), C.POINTER(aci_options)]
    lib.aci_elementwise_batch.argtypes = [C.POINTER(aci_job), C.c_int, C.c_int]
    lib.aci_workspace_query.argtypes = [C.POINTER(vp), C.c_int, C.c_int, C.c_int, vp, C.POINTER(C.c_size_t)]
    lib.aci_limits.argtypes = [ip, ip]
    lib.aci_prrlu.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int, C.c_int,
                              C.c_void_p, C.c_void_p, C.c_void_p, ip, dp, C.c_void_p]
    lib.aci_last_error.restype = C.c_char_p
    lib.aci_version.restype = C.c_char_p
    _lib = lib
    return lib


def _check(code):
    if code < 0:
        raise AciError(code, load().aci_last_error().decode())
    return code


def _dptr(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


class TensorTrain:
    """Device-resident TT handle (tt_t*). Cores are row-major [r_s][d_s][r_{s+1}]."""

    def __init__(self, handle):
        self._h = C.c_void_p(handle) if not isinstance(handle, C.c_void_p) else handle

    @classmethod
    def from_cores(cls, cores) -> "TensorTrain":
        """Real cores -> tt_create; complex cores (numpy complex128, interleaved) -> tt_create_z."""
        cores = list(cores.cores if hasattr(cores, "cores") else cores)
        cplx = any(np.iscomplexobj(c) for c in cores)
        dt = np.complex128 if cplx else np.float64
        cores = [np.ascontiguousarray(c, dtype=dt) for c in cores]
        L = len(cores)
        d = np.array([c.shape[1] for c in cores], np.int32)
        r = np.array([cores[0].shape[0]] + [c.shape[2] for c in cores], np.int32)
        ptrs = (C.POINTER(C.c_double) * L)(*[_dptr(c) for c in cores])
        h = C.c_void_p()
        fn = load().tt_create_z if cplx else load().tt_create
        _check(fn(L, d.ctypes.data_as(C.POINTER(C.c_int)), r.ctypes.data_as(C.POINTER(C.c_int)), ptrs, C.byref(h)))
        return cls(h)

    @classmethod
    def from_device(cls, d, ranks, dev_ptr: int, stream: int = 0) -> "TensorTrain":
        d = np.asarray(d, np.int32)
        r = np.asarray(ranks, np.int32)
        h = C.c_void_p()
        _check(load().tt_create_device(len(d), d.ctypes.data_as(C.POINTER(C.c_int)),
                                       r.ctypes.data_as(C.POINTER(C.c_int)), C.c_void_p(dev_ptr),
                                       C.c_void_p(stream), C.byref(h)))
        return cls(h)

    @property
    def handle(self):
        return self._h

    def shape(self):
        L = C.c_int()
        _check(load().tt_shape(self._h, C.byref(L), None, None))
        d = np.zeros(L.value, np.int32)
        r = np.zeros(L.value + 1, np.int32)
        _check(load().tt_shape(self._h, C.byref(L), d.ctypes.data_as(C.POINTER(C.c_int)),
                               r.ctypes.data_as(C.POINTER(C.c_int))))
        return [int(x) for x in d], [int(x) for x in r]

    @property
    def is_complex(self) -> bool:
        return bool(load().tt_is_complex(self._h))

    def cores(self):
        d, r = self.shape()
        dt = np.complex128 if self.is_complex else np.float64
        out = [np.zeros((r[s], d[s], r[s + 1]), dt) for s in range(len(d))]
        ptrs = (C.POINTER(C.c_double) * len(d))(*[_dptr(c) for c in out])
        _check(load().tt_get_cores(self._h, ptrs))
        return out

    def device_ptr(self) -> int:
        return load().tt_device_cores(self._h)

    def evaluate(self, idx) -> np.ndarray:
        idx = np.ascontiguousarray(idx, dtype=np.uint8)
        out = np.zeros(idx.shape[0], np.complex128 if self.is_complex else np.float64)
        _check(load().tt_evaluate(self._h, idx.shape[0], idx.ctypes.data, _dptr(out)))
        return out

    def evaluate_device(self, npts: int, dev_idx: int, dev_out: int, stream: int = 0):
        _check(load().tt_evaluate_device(self._h, npts, C.c_void_p(dev_idx), C.c_void_p(dev_out),
                                         C.c_void_p(stream)))

    def free(self):
        if self._h is not None and self._h.value:
            load().tt_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def _make_op(op, n_inputs):
    coef = np.ascontiguousarray(op["coef"], dtype=np.float64)
    expo = np.ascontiguousarray(op["expo"], dtype=np.int32).reshape(len(coef), n_inputs)
    return aci_op(len(coef), _dptr(coef), expo.ctypes.data_as(C.POINTER(C.c_int))), (coef, expo)


def _make_log(L, maxrank, max_sweeps):
    """An aci_pivot_log sized for max_sweeps iterations, and a reader returning
    {"log": [per-update dicts], "canon_cols": {s: columns}} once the call has returned."""
    cap_u = 2 * (L - 1) * max_sweeps
    cap_p = maxrank
    info = np.zeros((cap_u, 5), np.int32)
    es = np.zeros((cap_u, 2))
    rows = np.zeros((cap_u, cap_p), np.int32)
    cols = np.zeros((cap_u, cap_p), np.int32)
    cn = np.zeros(L + 1, np.int32)
    cc = np.zeros((L + 1, cap_p), np.int32)
    lg = aci_pivot_log(cap_u, cap_p, info.ctypes.data_as(C.POINTER(C.c_int)), _dptr(es),
                       rows.ctypes.data_as(C.POINTER(C.c_int)), cols.ctypes.data_as(C.POINTER(C.c_int)), 0,
                       cn.ctypes.data_as(C.POINTER(C.c_int)), cc.ctypes.data_as(C.POINTER(C.c_int)))

    def read():
        nw = lg.n_written
        return {"log": [{"bond": int(info[u, 0]), "dir": int(info[u, 1]), "rl": int(info[u, 2]),
                         "rr": int(info[u, 3]), "r": int(info[u, 4]), "eps": float(es[u, 0]),
                         "scale": float(es[u, 1]), "rows": rows[u, :info[u, 4]].copy(),
                         "cols": cols[u, :info[u, 4]].copy()} for u in range(nw)],
                "canon_cols": {s: cc[s, :cn[s]].copy() for s in range(1, L)}}

    read.keep = (info, es, rows, cols, cn, cc)
    return lg, read


def aci_elementwise(op, inputs, tol, maxrank, max_sweeps, y_init=None, seed=0, tol_mode=TOL_RELATIVE,
                    log=False, stream=0, workspace=None, index_sets=False, profile=False, iter_times=False,
                    concurrent=False, pivoting="full"):
    """Run aci_elementwise_ex. ``inputs`` are TensorTrain handles (aliases allowed).

    Returns (TensorTrain, status, report dict, extras dict).
    """
    lib = load()
    n = len(inputs)
    cop, keep = _make_op(op, n)
    hs = (C.c_void_p * n)(*[x.handle.value for x in inputs])
    out = C.c_void_p()
    rep = aci_report()
    opts = aci_options()
    opts.seed = seed
    opts.y_init = y_init.handle.value if y_init is not None else None
    opts.tol_mode = tol_mode
    opts.stream = stream or None
    opts.concurrent = 1 if concurrent else 0
    opts.pivoting = _PIVOTING[pivoting]
    extras = {}
    if workspace is not None:
        opts.workspace, opts.workspace_bytes = workspace
    if profile:
        prof = aci_profile()
        opts.profile = C.pointer(prof)
    if iter_times:
        iter_ms = np.zeros(max_sweeps, np.float32)
        opts.iter_ms = iter_ms.ctypes.data_as(C.POINTER(C.c_float))
    L = len(inputs[0].shape()[0])
    if log:
        lg, read_log = _make_log(L, maxrank, max_sweeps)
        opts.log = C.pointer(lg)
    if index_sets:
        Ibufs = [np.zeros((maxrank, b + 1), np.uint8) for b in range(L - 1)]
        Jbufs = [np.zeros((maxrank, max(L - s, 1)), np.uint8) for s in range(L + 1)]
        Ip = (C.POINTER(C.c_uint8) * L)(*[b.ctypes.data_as(C.POINTER(C.c_uint8)) for b in Ibufs],
                                        C.POINTER(C.c_uint8)())
        Jp = (C.POINTER(C.c_uint8) * (L + 1))(*[b.ctypes.data_as(C.POINTER(C.c_uint8)) for b in Jbufs])
        opts.I_sets = C.cast(Ip, C.POINTER(C.POINTER(C.c_uint8)))
        opts.J_sets = C.cast(Jp, C.POINTER(C.POINTER(C.c_uint8)))
    st = lib.aci_elementwise_ex(cop, hs, n, float(tol), int(maxrank), int(max_sweeps), C.byref(out), C.byref(rep),
                                C.byref(opts))
    _check(st)
    res = TensorTrain(out)
    if profile:
        extras["profile"] = prof.as_dict()
    if iter_times:
        extras["iter_ms"] = [float(x) for x in iter_ms[:rep.iterations]]
    if log:
        extras.update(read_log())
    if index_sets:
        _, rk = res.shape()
        extras["I"] = [Ibufs[b][:rk[b + 1]].copy() for b in range(L - 1)]
        extras["J"] = {s: Jbufs[s][:rk[s]].copy() for s in range(1, L)}
    return res, st, rep.as_dict(), extras


class aci_job(C.Structure):
    _fields_ = [("op", aci_op), ("inputs", C.POINTER(C.c_void_p)), ("n_inputs", C.c_int), ("tol", C.c_double),
                ("maxrank", C.c_int), ("max_sweeps", C.c_int), ("options", C.POINTER(aci_options)),
                ("out", C.POINTER(C.c_void_p)), ("rep", C.POINTER(aci_report)), ("status", C.c_int)]


def aci_elementwise_batch(jobs, max_parallel=0):
    """Run aci_elementwise_batch: ``jobs`` is a list of dicts with the aci_elementwise arguments
    (op, inputs, tol, maxrank, max_sweeps; optional y_init, seed, tol_mode, log). The products run
    concurrently on library threads and streams. Returns a list of (TensorTrain, status, report)
    in job order — (TensorTrain, status, report, extras) for jobs with log=True — and raises
    AciError if any job failed."""
    lib = load()
    n = len(jobs)
    arr = (aci_job * n)()
    keep, outs, reps, opts, readers = [], [], [], [], []
    for i, j in enumerate(jobs):
        ins = j["inputs"]
        cop, k = _make_op(j["op"], len(ins))
        hs = (C.c_void_p * len(ins))(*[x.handle.value for x in ins])
        o = aci_options()
        o.seed = j.get("seed", 0)
        o.y_init = j["y_init"].handle.value if j.get("y_init") is not None else None
        o.tol_mode = j.get("tol_mode", TOL_RELATIVE)
        o.pivoting = _PIVOTING[j.get("pivoting", "full")]
        if j.get("log"):
            lg, rd = _make_log(len(ins[0].shape()[0]), int(j["maxrank"]), int(j["max_sweeps"]))
            o.log = C.pointer(lg)
            keep += [lg, rd]
            readers.append(rd)
        else:
            readers.append(None)
        out = C.c_void_p()
        rep = aci_report()
        keep += [cop, k, hs]
        outs.append(out)
        reps.append(rep)
        opts.append(o)
        arr[i].op = cop
        arr[i].inputs = C.cast(hs, C.POINTER(C.c_void_p))
        arr[i].n_inputs = len(ins)
        arr[i].tol = float(j["tol"])
        arr[i].maxrank = int(j["maxrank"])
        arr[i].max_sweeps = int(j["max_sweeps"])
        arr[i].options = C.pointer(o)
        arr[i].out = C.pointer(out)
        arr[i].rep = C.pointer(rep)
    st = lib.aci_elementwise_batch(arr, n, int(max_parallel))
    res = [(TensorTrain(outs[i]) if outs[i].value else None, int(arr[i].status), reps[i].as_dict())
           + ((readers[i](),) if readers[i] is not None else ()) for i in range(n)]
    if st < 0:
        for r in res:
            if r[0] is not None:
                r[0].free()
    _check(st)
    return res


def workspace_query(inputs, maxrank, y_init=None, max_sweeps=64) -> int:
    n = len(inputs)
    hs = (C.c_void_p * n)(*[x.handle.value for x in inputs])
    b = C.c_size_t()
    _check(load().aci_workspace_query(hs, n, maxrank, max_sweeps, y_init.handle.value if y_init is not None else None,
                                      C.byref(b)))
    return b.value


def prrlu(M, maxrank: int, tol: float = 0.0, relative: bool = True, static=(0, 0), want_u: bool = True,
          stream=None) -> dict:
    """a5 alone (include/aci.h aci_prrlu) on a device copy of the float64 block M (torch CUDA tensor
    or numpy array): rows, cols (selection order), U (r x n), eps. Argument marshalling only."""
    import torch
    Mt = torch.as_tensor(M, dtype=torch.float64).cuda().contiguous()
    m, n = Mt.shape
    k = max(1, min(maxrank, m, n))
    rows = torch.full((k,), -1, dtype=torch.int32, device=Mt.device)
    cols = torch.full((k,), -1, dtype=torch.int32, device=Mt.device)
    U = torch.zeros((k, n), dtype=torch.float64, device=Mt.device) if want_u else None
    r, e = C.c_int(), C.c_double()
    st = stream if stream is not None else torch.cuda.current_stream().cuda_stream
    _check(load().aci_prrlu(Mt.data_ptr(), m, n, maxrank, tol, 0 if relative else 1, int(static[0]), int(static[1]),
                            rows.data_ptr(), cols.data_ptr(), U.data_ptr() if U is not None else None, C.byref(r),
                            C.byref(e), st))
    rr = r.value
    out = {"r": rr, "rows": rows[:rr].cpu().numpy(), "cols": cols[:rr].cpu().numpy(), "eps": e.value}
    if U is not None:
        out["U"] = U[:rr].cpu().numpy()
    return out


def limits():
    a, b = C.c_int(), C.c_int()
    _check(load().aci_limits(C.byref(a), C.byref(b)))
    return a.value, b.value


def version() -> str:
    return load().aci_version().decode()
