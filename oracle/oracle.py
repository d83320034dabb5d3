"""ctypes face of the CPU checkers.  TEST INFRASTRUCTURE ONLY.

Two interchangeable back ends with one ABI (oracle/farqb_oracle.h):

* ``Oracle("port")``      -- lib/libfarqb_oracle.so, the plain-C restatement of the
                             reference algorithm (always buildable: ``make -C oracle``).
* ``Oracle("reference")`` -- _ref/librsvd_ref.so, the UNMODIFIED reference sources
                             compiled in place plus ref_shim.cpp (``make -C oracle ref``;
                             needs /root/reference at build time only).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this module; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_LIB = os.path.join(HERE, "lib", "libfarqb_oracle.so")
REF_LIB = os.path.join(HERE, "_ref", "librsvd_ref.so")

GAUSSIAN, BERNOULLI, STD_BERNOULLI, SPARSE_SIGN, SPARSE_GAUSSIAN = range(5)
OK, ERR_CONFIG, ERR_DIMENSION, ERR_BLOCK_DEGENERATE, ERR_TOLERANCE = 0, 1, 2, 3, 4


class Block(C.Structure):
    _fields_ = [
        ("is_dense", C.c_int), ("rows", C.c_int), ("cols", C.c_int),
        ("dense", C.POINTER(C.c_double)), ("col_ptr", C.POINTER(C.c_int)),
        ("row_idx", C.POINTER(C.c_int)), ("values", C.POINTER(C.c_double)),
        ("nnz", C.c_int64), ("centered", C.c_int), ("p", C.c_double),
        ("std_scale", C.c_double),
    ]


class Config(C.Structure):
    _fields_ = [
        ("eps", C.c_double), ("power", C.c_int), ("block", C.c_int), ("kind", C.c_int),
        ("p", C.c_double), ("seed", C.c_uint64), ("zeta", C.c_int), ("max_iters", C.c_int),
        ("shift_convention", C.c_int), ("relative", C.c_int),
    ]


class Result(C.Structure):
    _fields_ = [
        ("status", C.c_int), ("m", C.c_int), ("n", C.c_int), ("rank", C.c_int),
        ("blocks", C.c_int), ("converged", C.c_int), ("residual_sq", C.c_double),
        ("norm_a_sq", C.c_double), ("sigma", C.POINTER(C.c_double)),
        ("u", C.POINTER(C.c_double)), ("v", C.POINTER(C.c_double)),
        ("block_residuals", C.POINTER(C.c_double)), ("block_ids", C.POINTER(C.c_int)),
        ("n_ids", C.c_int), ("resolved_block", C.c_int), ("resolved_max_iters", C.c_int),
        ("resolved_p", C.c_double), ("message", C.c_char * 256),
    ]


SOURCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_int, C.POINTER(Block))


@dataclass
class SketchArrays:
    """One Omega block as numpy arrays (dense or CSC)."""
    is_dense: bool
    rows: int
    cols: int
    dense: np.ndarray | None = None       # rows x cols, Fortran order
    col_ptr: np.ndarray | None = None
    row_idx: np.ndarray | None = None
    values: np.ndarray | None = None
    centered: bool = False
    p: float = 0.0
    std_scale: float = 0.0

    def densify(self) -> np.ndarray:
        if self.is_dense:
            return self.dense
        d = np.zeros((self.rows, self.cols), order="F")
        for j in range(self.cols):
            s, e = self.col_ptr[j], self.col_ptr[j + 1]
            d[self.row_idx[s:e], j] = self.values[s:e]
        return d


@dataclass
class RunResult:
    status: int
    rank: int
    blocks: int
    converged: bool
    residual_sq: float
    norm_a_sq: float
    sigma: np.ndarray
    u: np.ndarray | None
    v: np.ndarray | None
    block_residuals: np.ndarray
    block_ids: list
    resolved_block: int
    resolved_max_iters: int
    resolved_p: float
    message: str = ""
    extra: dict = field(default_factory=dict)


def _ensure_built(path: str, target: str) -> None:
    if os.path.exists(path):
        return
    subprocess.run(["make", "-s", "-C", HERE, target], check=True)


def reference_available() -> bool:
    return os.path.exists(REF_LIB) or os.path.isdir("/root/reference/proj/src")


class Oracle:
    def __init__(self, which: str = "port"):
        self.which = which
        if which == "port":
            _ensure_built(PORT_LIB, "all")
            self.lib = C.CDLL(PORT_LIB)
            pre = "fqo_"
        elif which == "reference":
            _ensure_built(REF_LIB, "ref")
            self.lib = C.CDLL(REF_LIB)
            pre = "ref_"
        else:
            raise ValueError(which)
        L = self.lib
        self._pre = pre
        g = lambda name: getattr(L, pre + name)
        for name in ("philox_u32",):
            g(name).argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_int, C.POINTER(C.c_uint32)]
        for name in ("philox_units", "philox_gaussians"):
            g(name).argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_int, C.POINTER(C.c_double)]
        g("gen_sketch").argtypes = [C.c_int, C.c_double, C.c_uint64, C.c_int, C.c_int, C.c_int,
                                    C.c_int, C.POINTER(Block)]
        g("gen_sketch").restype = C.c_int
        g("block_free").argtypes = [C.POINTER(Block)]
        g("sparse_dense_mul").argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p,
                                          C.c_void_p, C.c_int, C.c_void_p]
        g("centering_column").argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_double, C.c_void_p]
        g("run_fixed_precision").argtypes = [C.c_void_p, C.c_int, C.c_int, C.POINTER(Config),
                                             SOURCE_FN, C.c_void_p, C.c_int, C.POINTER(Result)]
        g("run_fixed_rank").argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.POINTER(Config),
                                        SOURCE_FN, C.c_void_p, C.c_int, C.POINTER(Result)]
        g("result_free").argtypes = [C.POINTER(Result)]
        if which == "reference":
            L.ref_run_traced.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int,
                                         C.POINTER(Config), SOURCE_FN, C.c_void_p, C.c_int,
                                         C.POINTER(Result)]
            L.ref_gen_synthetic.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_void_p]
            L.ref_random_orthonormal.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_uint32, C.c_void_p]
            L.ref_load_matrix.argtypes = [C.c_char_p, C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                          C.POINTER(C.POINTER(C.c_double)), C.c_char_p, C.c_int,
                                          C.POINTER(C.c_longlong)]
            L.ref_save_matrix.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_char_p, C.c_char_p, C.c_char_p,
                                          C.c_int]
            L.ref_free.argtypes = [C.c_void_p]
            L.ref_run_experiment.argtypes = [C.c_char_p, C.c_char_p, C.c_int]
            L.ref_check_experiment_config.argtypes = [C.c_char_p, C.c_char_p, C.c_int]
            L.ref_read_report_csv.argtypes = [C.c_char_p, C.c_char_p, C.c_int, C.POINTER(C.c_longlong)]
        else:
            L.fqo_gemm_nn.argtypes = [C.c_int] * 3 + [C.c_void_p, C.c_int, C.c_void_p, C.c_int,
                                                      C.c_void_p, C.c_int]
            L.fqo_gemm_tn.argtypes = L.fqo_gemm_nn.argtypes
            L.fqo_frob_norm_sq.argtypes = [C.c_void_p, C.c_int64]
            L.fqo_frob_norm_sq.restype = C.c_double
            L.fqo_sym_eig.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
            L.fqo_chol_factor.argtypes = [C.c_void_p, C.c_int, C.c_double, C.c_double, C.c_void_p]

    def _fn(self, name):
        return getattr(self.lib, self._pre + name)

    # ---- RNG ------------------------------------------------------------------
    def philox_u32(self, seed, block_id, column, count):
        out = np.zeros(count, dtype=np.uint32)
        self._fn("philox_u32")(seed, block_id, column, count,
                               out.ctypes.data_as(C.POINTER(C.c_uint32)))
        return out

    def philox_units(self, seed, block_id, column, count):
        out = np.zeros(count)
        self._fn("philox_units")(seed, block_id, column, count,
                                 out.ctypes.data_as(C.POINTER(C.c_double)))
        return out

    def philox_gaussians(self, seed, block_id, column, count):
        out = np.zeros(count)
        self._fn("philox_gaussians")(seed, block_id, column, count,
                                     out.ctypes.data_as(C.POINTER(C.c_double)))
        return out

    # ---- sketches ---------------------------------------------------------------
    def gen_sketch(self, kind, p, seed, n, l, block_id, zeta=0) -> SketchArrays:
        blk = Block()
        rc = self._fn("gen_sketch")(kind, p, seed, zeta, n, l, block_id, C.byref(blk))
        if rc != 0:
            raise ValueError(f"gen_sketch failed with status {rc}")
        try:
            return _block_to_arrays(blk)
        finally:
            self._fn("block_free")(C.byref(blk))

    def sparse_dense_mul(self, a: np.ndarray, s: SketchArrays) -> np.ndarray:
        a = np.asfortranarray(a, dtype=np.float64)
        m, n = a.shape
        c = np.zeros((m, s.cols), order="F")
        cp = np.ascontiguousarray(s.col_ptr, dtype=np.int32)
        ri = np.ascontiguousarray(s.row_idx, dtype=np.int32)
        va = np.ascontiguousarray(s.values, dtype=np.float64)
        self._fn("sparse_dense_mul")(a.ctypes.data, m, n, cp.ctypes.data, ri.ctypes.data,
                                     va.ctypes.data, s.cols, c.ctypes.data)
        return c

    def centering_column(self, a: np.ndarray, p: float) -> np.ndarray:
        a = np.asfortranarray(a, dtype=np.float64)
        z = np.zeros(a.shape[0])
        self._fn("centering_column")(a.ctypes.data, a.shape[0], a.shape[1], p, z.ctypes.data)
        return z

    # ---- driver ---------------------------------------------------------------
    def run(self, a, *, eps=0.0, power=0, block=0, kind=GAUSSIAN, p=0.0, seed=0, zeta=0,
            max_iters=0, shift_convention=0, relative=True, rank=None, source=None,
            want_vectors=False, traced=False) -> RunResult:
        """run_fixed_precision (rank None) or run_fixed_rank.

        ``source(n, b, block_id) -> SketchArrays`` injects Omega blocks exactly as the
        reference's BlockSource does (driver.hpp:67-73)."""
        a = np.asfortranarray(a, dtype=np.float64)
        m, n = a.shape
        cfg = Config(eps, power, block, kind, p, seed, zeta, max_iters, shift_convention,
                     int(relative))
        res = Result()
        keep = []
        err = []

        def cb(_user, nn, bb, bid, out):
            try:
                arr = source(nn, bb, bid)
                out[0] = _arrays_to_block(arr, keep)
                return 0
            except Exception as e:  # noqa: BLE001 - reported through the status
                err.append(e)
                return 1

        fn = SOURCE_FN(cb) if source is not None else SOURCE_FN()
        if traced:
            if self.which != "reference":
                raise ValueError("traced runs are a reference-shim feature")
            self.lib.ref_run_traced(a.ctypes.data, m, n, rank or 0, int(rank is None),
                                    C.byref(cfg), fn, None, int(want_vectors), C.byref(res))
        elif rank is None:
            self._fn("run_fixed_precision")(a.ctypes.data, m, n, C.byref(cfg), fn, None,
                                            int(want_vectors), C.byref(res))
        else:
            self._fn("run_fixed_rank")(a.ctypes.data, m, n, rank, C.byref(cfg), fn, None,
                                       int(want_vectors), C.byref(res))
        if err:
            raise err[0]
        try:
            r = res.rank
            sigma = np.ctypeslib.as_array(res.sigma, (r,)).copy() if r and res.sigma else np.zeros(0)
            u = v = None
            if want_vectors and r and res.u:
                u = np.ctypeslib.as_array(res.u, (r * m,)).reshape((m, r), order="F").copy()
                v = np.ctypeslib.as_array(res.v, (r * n,)).reshape((n, r), order="F").copy()
            nb = res.blocks
            br = (np.ctypeslib.as_array(res.block_residuals, (nb,)).copy()
                  if nb and res.block_residuals else np.zeros(0))
            ids = (list(np.ctypeslib.as_array(res.block_ids, (res.n_ids,)))
                   if res.n_ids and res.block_ids else [])
            return RunResult(res.status, r, res.blocks, bool(res.converged), res.residual_sq,
                             res.norm_a_sq, sigma, u, v, br, [int(i) for i in ids],
                             res.resolved_block, res.resolved_max_iters, res.resolved_p,
                             res.message.decode(errors="replace"))
        finally:
            self._fn("result_free")(C.byref(res))

    # ---- reference-only helpers -----------------------------------------------
    def gen_synthetic(self, kind: int, n: int, seed: int) -> np.ndarray:
        out = np.zeros((n, n), order="F")
        rc = self.lib.ref_gen_synthetic(kind, n, seed, out.ctypes.data)
        if rc != 0:
            raise ValueError("gen_synthetic failed")
        return out

    def random_orthonormal(self, n: int, r: int, seed: int, stream: int) -> np.ndarray:
        out = np.zeros((n, r), order="F")
        rc = self.lib.ref_random_orthonormal(n, r, seed, stream, out.ctypes.data)
        if rc != 0:
            raise ValueError("random_orthonormal failed")
        return out


    # ---- matrix files / experiment driver (reference only) -------------------------
    # Errors come back as (status, message, offset): status 1 FormatError, 2 ConfigError,
    # 3 DimensionError, 4 other (ref_shim.cpp).
    def load_matrix(self, path, fmt):
        rows, cols, off = C.c_int(), C.c_int(), C.c_longlong(-1)
        data = C.POINTER(C.c_double)()
        err = C.create_string_buffer(512)
        st = self.lib.ref_load_matrix(os.fsencode(path), fmt.encode(), C.byref(rows), C.byref(cols),
                                      C.byref(data), err, 512, C.byref(off))
        if st:
            return None, (st, err.value.decode(), off.value)
        try:
            n = rows.value * cols.value
            flat = np.ctypeslib.as_array(data, shape=(max(n, 1),))[:n].copy()
        finally:
            self.lib.ref_free(data)
        return np.asfortranarray(flat.reshape((cols.value, rows.value)).T), None

    def save_matrix(self, a, path, fmt):
        a = np.asfortranarray(a, dtype=np.float64)
        err = C.create_string_buffer(512)
        st = self.lib.ref_save_matrix(a.ctypes.data, a.shape[0], a.shape[1], os.fsencode(path), fmt.encode(),
                                      err, 512)
        return None if st == 0 else (st, err.value.decode())

    def run_experiment(self, config_path):
        err = C.create_string_buffer(512)
        st = self.lib.ref_run_experiment(os.fsencode(config_path), err, 512)
        return None if st == 0 else (st, err.value.decode())

    def check_experiment_config(self, config_path):
        err = C.create_string_buffer(512)
        st = self.lib.ref_check_experiment_config(os.fsencode(config_path), err, 512)
        return None if st == 0 else (st, err.value.decode())

    def read_report_csv(self, path):
        err, off = C.create_string_buffer(512), C.c_longlong(-1)
        n = self.lib.ref_read_report_csv(os.fsencode(path), err, 512, C.byref(off))
        return (n, None) if n >= 0 else (None, (-n, err.value.decode(), off.value))


def _block_to_arrays(blk: Block) -> SketchArrays:
    if blk.is_dense:
        d = np.ctypeslib.as_array(blk.dense, (blk.rows * blk.cols,)).reshape(
            (blk.rows, blk.cols), order="F").copy()
        return SketchArrays(True, blk.rows, blk.cols, dense=d, p=blk.p)
    nnz = int(blk.nnz)
    cp = np.ctypeslib.as_array(blk.col_ptr, (blk.cols + 1,)).copy()
    ri = np.ctypeslib.as_array(blk.row_idx, (max(nnz, 1),))[:nnz].copy()
    va = np.ctypeslib.as_array(blk.values, (max(nnz, 1),))[:nnz].copy()
    return SketchArrays(False, blk.rows, blk.cols, col_ptr=cp, row_idx=ri, values=va,
                        centered=bool(blk.centered), p=blk.p, std_scale=blk.std_scale)


def _arrays_to_block(s: SketchArrays, keep: list) -> Block:
    blk = Block()
    blk.is_dense = int(s.is_dense)
    blk.rows, blk.cols = s.rows, s.cols
    blk.centered = int(s.centered)
    blk.p = s.p
    blk.std_scale = s.std_scale
    if s.is_dense:
        d = np.asfortranarray(s.dense, dtype=np.float64)
        keep.append(d)
        blk.dense = d.ctypes.data_as(C.POINTER(C.c_double))
    else:
        cp = np.ascontiguousarray(s.col_ptr, dtype=np.int32)
        ri = np.ascontiguousarray(s.row_idx, dtype=np.int32)
        va = np.ascontiguousarray(s.values, dtype=np.float64)
        if ri.size == 0:
            ri = np.zeros(1, np.int32)
            va = np.zeros(1)
        keep.extend([cp, ri, va])
        blk.col_ptr = cp.ctypes.data_as(C.POINTER(C.c_int))
        blk.row_idx = ri.ctypes.data_as(C.POINTER(C.c_int))
        blk.values = va.ctypes.data_as(C.POINTER(C.c_double))
        blk.nnz = int(s.col_ptr[-1])
    return blk
