"""Python mirror of the reference's QB API (rsvd::, /root/reference/proj/include/rsvd/).

Same names, argument meaning and error behaviour as the C++ reference, so a
caller of ``rsvd::run_fixed_precision(a, cfg, source)`` (driver.hpp:98-99) can
switch to ``run_fixed_precision(a, cfg, source)`` here; the difference is the
result, which carries the north-star QB outputs (Q, B', rank, error indicator)
computed by the sm_100a engine in libfarqb.so:

  reference                                this module
  ---------------------------------------  ------------------------------------
  SketchKind, sketch_kind_name/_from_name  SketchKind, sketch_kind_name/_from_name
  SketchSpec{kind, p, seed}                SketchSpec(kind, p, seed, zeta=0)
  FarpcaConfig{eps, power, block, sketch,  FarpcaConfig(...)  same fields
    max_iters, shift_convention, relative}
  ShiftConvention                          ShiftConvention
  BlockSource::next(n, b, block_id)        BlockSource.next(n, b, block_id) -> SketchBlock
  SketchBlock / SparseSketch               SketchBlock (numpy arrays)
  run_fixed_precision / run_fixed_rank     run_fixed_precision / run_fixed_rank -> QBResult
  gen_sketch                               gen_sketch (generated on the device)
  ConfigError, DimensionError,             same exception classes
  BlockDegenerate, ToleranceNotReached,
  ConvergenceFailure
  default_density/_block/_max_iters        same

Matrices are column-major (Fortran order) float64, like DenseMatrix
(dense_matrix.hpp:13-51).  Accepted inputs: numpy arrays (host), torch tensors
on the host or on a CUDA device.  Every compute call runs on the GPU; without
one the calls raise CudaError.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _native as N

# ---------------------------------------------------------------- errors ----


class RsvdError(Exception):
    status = -1


class ConfigError(RsvdError, ValueError):
    status = 1


class DimensionError(RsvdError, ValueError):
    status = 2


class BlockDegenerate(RsvdError, RuntimeError):
    """errors.hpp:28-37; carries the accepted block count and residual."""
    status = 3

    def __init__(self, msg, blocks_accepted=0, residual_sq=0.0, norm_a_sq=0.0):
        super().__init__(msg)
        self.blocks_accepted = blocks_accepted
        self.residual_sq = residual_sq
        self.norm_a_sq = norm_a_sq


class ToleranceNotReached(RsvdError, RuntimeError):
    """driver.hpp:60-65; ``partial`` is the QB result after max_iters blocks."""
    status = 4

    def __init__(self, msg, partial=None):
        super().__init__(msg)
        self.partial = partial


class CudaError(RsvdError, RuntimeError):
    status = 5


class InvalidArgument(RsvdError, ValueError):
    status = 7


class ConvergenceFailure(RsvdError, RuntimeError):
    status = 8


class CallbackError(RsvdError, RuntimeError):
    status = 9


class AllocError(RsvdError, MemoryError):
    status = 10


_ERRORS = {c.status: c for c in (ConfigError, DimensionError, BlockDegenerate, ToleranceNotReached,
                                 CudaError, InvalidArgument, ConvergenceFailure, CallbackError,
                                 AllocError)}


def _raise(status: int, what: str = ""):
    msg = N.lib().fqb_last_error().decode(errors="replace")
    cls = _ERRORS.get(status, RsvdError)
    raise cls(f"{what}: {msg}" if what else msg)


# ------------------------------------------------------------------ types ---


class SketchKind(enum.IntEnum):
    Gaussian = 0
    Bernoulli = 1
    StdBernoulli = 2
    SparseSign = 3
    SparseGaussian = 4


_KIND_NAMES = {SketchKind.Gaussian: "gaussian", SketchKind.Bernoulli: "bernoulli",
               SketchKind.StdBernoulli: "stdbernoulli", SketchKind.SparseSign: "sparsesign",
               SketchKind.SparseGaussian: "sparsegaussian"}


def sketch_kind_name(k: SketchKind) -> str:
    return _KIND_NAMES.get(SketchKind(k), "unknown")


def sketch_kind_from_name(name: str) -> SketchKind:
    for k, v in _KIND_NAMES.items():
        if v == name:
            return k
    raise ConfigError(f"unknown sketch kind: {name}")


class ShiftConvention(enum.IntEnum):
    LastDiagonal = 0
    FirstDiagonal = 1


@dataclass
class SketchSpec:
    kind: SketchKind = SketchKind.Gaussian
    p: float = 0.0
    seed: int = 0
    zeta: int = 0     # > 0: exactly zeta nonzeros per column (sparse sign / Gaussian)


@dataclass
class FarpcaConfig:
    eps: float = 0.0
    power: int = 0
    block: int = 0
    sketch: SketchSpec = field(default_factory=SketchSpec)
    max_iters: int = 0
    shift_convention: ShiftConvention = ShiftConvention.LastDiagonal
    relative: bool = False

    def _c(self) -> N.ConfigC:
        s = self.sketch
        return N.ConfigC(float(self.eps), int(self.power), int(self.block),
                         N.SketchSpecC(int(s.kind), float(s.p), int(s.seed) & (2**64 - 1), int(s.zeta)),
                         int(self.max_iters), int(self.shift_convention), int(bool(self.relative)))


@dataclass
class SketchBlock:
    """rsvd::SketchBlock (sketch.hpp:37-44) with numpy arrays."""
    is_dense: bool
    rows: int
    cols: int
    dense: Optional[np.ndarray] = None      # rows x cols, Fortran order
    col_ptr: Optional[np.ndarray] = None
    row_idx: Optional[np.ndarray] = None
    values: Optional[np.ndarray] = None
    centered: bool = False
    p: float = 0.0
    std_scale: float = 0.0

    @property
    def nnz(self) -> int:
        return 0 if self.is_dense else int(self.col_ptr[-1])

    def densify(self) -> np.ndarray:
        if self.is_dense:
            return self.dense
        d = np.zeros((self.rows, self.cols), order="F")
        for j in range(self.cols):
            s, e = self.col_ptr[j], self.col_ptr[j + 1]
            d[self.row_idx[s:e], j] = self.values[s:e]
        return d


class BlockSource:
    """rsvd::BlockSource (driver.hpp:67-73): supplies the raw block for (n, b, block_id)."""

    def next(self, n: int, b: int, block_id: int) -> SketchBlock:  # pragma: no cover - interface
        raise NotImplementedError


@dataclass
class QBResult:
    """QB factorization A ~ Q B with the reference's ApproxSvd scalars.

    q  : m x rank, orthonormal columns
    bt : n x rank, B transposed (B = Q' A is rank x n)
    residual_sq : the error indicator E = ||A||_F^2 - sum ||B_j||_F^2
    """
    q: object
    bt: object
    rank: int
    blocks: int
    converged: bool
    residual_sq: float
    norm_a_sq: float
    block_residuals: np.ndarray
    block_ids: list
    resolved_block: int
    resolved_max_iters: int
    resolved_p: float
    elapsed_ms: float
    gpu_launches: int
    # rsvd::ApproxSvd fields (driver.hpp:45-58), present when svd=True
    u: object = None
    sigma: Optional[np.ndarray] = None
    v: object = None
    v_flagged: Optional[np.ndarray] = None
    svd_residual_sq: Optional[float] = None

    @property
    def b(self):
        return None if self.bt is None else self.bt.T

    def svd_rank(self) -> int:
        return 0 if self.sigma is None else len(self.sigma)


def default_density(kind: SketchKind, n: int) -> float:
    return N.lib().fqb_default_density(int(kind), int(n))


def default_block(m: int, n: int) -> int:
    return N.lib().fqb_default_block(int(m), int(n))


def default_max_iters(n: int, b: int) -> int:
    return N.lib().fqb_default_max_iters(int(n), int(b))


# ----------------------------------------------------------------- engine ---


class _DeviceBuffer:
    """Owns a library-allocated device array; exposes __cuda_array_interface__."""

    def __init__(self, ptr: int, rows: int, cols: int, ld: int):
        self.ptr = ptr
        self.__cuda_array_interface__ = {
            "shape": (cols, rows), "strides": (ld * 8, 8), "typestr": "<f8",
            "data": (ptr, False), "version": 3}

    def __del__(self):
        try:
            import torch  # noqa: F401
            from . import _native
            _cudart_free(self.ptr)
        except Exception:  # noqa: BLE001 - interpreter shutdown
            pass


class _HostBuffer:
    """Owns a library-allocated pinned host array (fqb_host_free on release); a
    column-major rows x cols float64 view via __array_interface__ -- no copy."""

    def __init__(self, ptr: int, rows: int, cols: int):
        self.ptr = ptr
        self.__array_interface__ = {
            "shape": (rows, cols), "strides": (8, rows * 8), "typestr": "<f8",
            "data": (ptr, False), "version": 3}

    def __del__(self):
        try:
            N.lib().fqb_host_free(self.ptr)
        except Exception:  # noqa: BLE001 - interpreter shutdown
            pass


def _host_array(ptr: int, rows: int, cols: int) -> np.ndarray:
    return np.asarray(_HostBuffer(ptr, rows, cols))


def _cudart_free(ptr: int) -> None:
    r = N.ResultC()
    r.on_device = 1
    r.q = ptr
    r.bt = None
    N.lib().fqb_result_free(C.byref(r))


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def _as_colmajor(a):
    """-> (pointer, m, n, lda, on_device, keepalive, is_f32).

    float64 runs the FP64 engine; float32 selects the FP32 input mode (A kept in
    FP32 on the device, every product in FP64 -- fqb_qb_*_f32)."""
    if _is_torch(a):
        import torch
        if a.dtype not in (torch.float64, torch.float32) or a.dim() != 2:
            raise InvalidArgument("A must be a 2-D float64 or float32 tensor")
        m, n = a.shape
        if not (a.stride(0) == 1 and (a.stride(1) >= max(m, 1) or n == 1)):
            a = a.t().contiguous().t()  # column-major copy
        lda = a.stride(1) if n > 1 else max(m, 1)
        return a.data_ptr(), m, n, lda, a.is_cuda, a, a.dtype == torch.float32
    src = np.asarray(a)
    dt = np.float32 if src.dtype == np.float32 else np.float64
    arr = np.asfortranarray(src, dtype=dt)
    if arr.ndim != 2:
        raise InvalidArgument("A must be 2-D")
    m, n = arr.shape
    return arr.ctypes.data, m, n, max(m, 1), False, arr, dt == np.float32


class SlicedOperand:
    """A matrix held as Ozaki slices on the device (both layouts); products with
    up to 64 right-hand columns run on the INT8 tensor cores (fqb_sliced_gemm)."""

    def __init__(self, engine, handle, m, n):
        self._eng, self._s, self.m, self.n = engine, handle, m, n

    def gemm(self, trans_a: bool, nb, alpha, b_ptr, ldb, beta, c_ptr, ldc):
        """C = alpha op(A) B + beta C; op(A) = A' if trans_a (C is n x nb) else A (C is m x nb)."""
        if self._s is None:
            raise InvalidArgument("sliced operand was freed")
        st = self._eng._lib.fqb_sliced_gemm(self._eng._h, self._s, int(trans_a), nb, alpha, b_ptr, ldb, beta,
                                            c_ptr, ldc)
        if st:
            _raise(st, "fqb_sliced_gemm")

    def gemm_again(self, alpha, beta, c_ptr, ldc):
        """The last gemm() once more on the B slices it left (nb <= 128): only the tensor-core
        GEMM kernel runs (fqb_sliced_gemm_again)."""
        if self._s is None:
            raise InvalidArgument("sliced operand was freed")
        st = self._eng._lib.fqb_sliced_gemm_again(self._eng._h, self._s, alpha, beta, c_ptr, ldc)
        if st:
            _raise(st, "fqb_sliced_gemm_again")

    def gemm_mn(self, nb, alpha, b_ptr, ldb, beta, c_ptr, ldc):
        """C (m x nb) = alpha A B + beta C from the A'Y-layout slices read MN-major
        (fqb_sliced_gemm_mn; the engine's Y -= Q C)."""
        if self._s is None:
            raise InvalidArgument("sliced operand was freed")
        st = self._eng._lib.fqb_sliced_gemm_mn(self._eng._h, self._s, nb, alpha, b_ptr, ldb, beta, c_ptr, ldc)
        if st:
            _raise(st, "fqb_sliced_gemm_mn")

    def free(self):
        if self._s is not None:
            self._eng._lib.fqb_sliced_free(self._eng._h, self._s)
            self._s = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.free()

    def __del__(self):
        try:
            self.free()
        except Exception:  # pragma: no cover - interpreter teardown
            pass


class Engine:
    """One libfarqb handle (one device, one stream, reusable workspace)."""

    def __init__(self, device: int = 0):
        self._lib = N.lib()
        h = C.c_void_p()
        st = self._lib.fqb_create(int(device), C.byref(h))
        if st != 0:
            _raise(st, "fqb_create")
        self._h = h
        self.device = device

    def close(self):
        if getattr(self, "_h", None):
            self._lib.fqb_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass

    @property
    def launch_count(self) -> int:
        return self._lib.fqb_launch_count(self._h)

    @property
    def collective_count(self) -> int:
        return self._lib.fqb_collective_count(self._h)

    def set_pass_timing(self, on: bool = True) -> None:
        """Arm (and reset) the CUDA-event timing of the A-pass k_ozaki launches
        (fqb_set_pass_timing)."""
        st = self._lib.fqb_set_pass_timing(self._h, 1 if on else 0)
        if st:
            _raise(st, "fqb_set_pass_timing")

    def pass_timing(self) -> tuple[float, int, float]:
        """(summed launch ms, launches, algorithmic FP64 bytes) since set_pass_timing."""
        ms, n, by = C.c_double(), C.c_int64(), C.c_double()
        st = self._lib.fqb_pass_timing(self._h, C.byref(ms), C.byref(n), C.byref(by))
        if st:
            _raise(st, "fqb_pass_timing")
        return ms.value, n.value, by.value

    def attach_comm(self, group=None, backend: str = "nccl") -> None:
        """Row-sharded mode: subsequent runs take this rank's row block of A
        (see paper_2506_03859_b200.dist.partition_rows).  backend "nccl": the engine's
        own NCCL communicator over NVLink; "host": the reduction points go through
        torch.distributed on the host (any process group, e.g. gloo)."""
        from . import dist
        if backend == "host":
            dist.attach_host(self, group)
        else:
            dist.attach(self, group)

    def detach_comm(self) -> None:
        st = self._lib.fqb_comm_detach(self._h)
        if st:
            _raise(st, "fqb_comm_detach")

    def set_stream(self, stream_ptr: int | None):
        st = self._lib.fqb_set_stream(self._h, stream_ptr)
        if st:
            _raise(st, "fqb_set_stream")

    def synchronize(self):
        st = self._lib.fqb_synchronize(self._h)
        if st:
            _raise(st, "fqb_synchronize")

    # ---- the QB loop --------------------------------------------------------
    def run_fixed_precision(self, a, cfg: FarpcaConfig, source: BlockSource | None = None,
                            output: str = "device", svd: bool = False) -> QBResult:
        """svd=True also assembles U, sigma, V (rsvd::ApproxSvd, assemble_svd)."""
        return self._run(a, cfg, source, output, rank=None, svd=svd)

    def run_fixed_rank(self, a, rank: int, cfg: FarpcaConfig, source: BlockSource | None = None,
                       output: str = "device", svd: bool = False) -> QBResult:
        """svd=True returns exactly `rank` triplets (drop_smallest, driver.cpp:85-106)."""
        return self._run(a, cfg, source, output, rank=rank, svd=svd)

    def _run(self, a, cfg, source, output, rank, svd=False):
        ptr, m, n, lda, on_dev, keep, f32 = _as_colmajor(a)
        flags = {"device": N.OUT_DEVICE, "host": N.OUT_HOST, "none": N.OUT_NONE}[output]
        if svd:
            flags |= N.OUT_SVD
        res = N.ResultC()
        ccfg = cfg._c()
        cb, err, hold = self._make_source(source)
        fp = self._lib.fqb_qb_fixed_precision_f32 if f32 else self._lib.fqb_qb_fixed_precision
        fr = self._lib.fqb_qb_fixed_rank_f32 if f32 else self._lib.fqb_qb_fixed_rank
        if rank is None:
            st = fp(self._h, ptr, m, n, lda, int(on_dev), C.byref(ccfg), cb, None, flags, C.byref(res))
        else:
            st = fr(self._h, ptr, m, n, lda, int(on_dev), int(rank), C.byref(ccfg), cb, None, flags, C.byref(res))
        del keep, hold
        if err:
            self._lib.fqb_result_free(C.byref(res))
            raise CallbackError("block source raised") from err[0]
        if st not in (0, 3, 4):
            self._lib.fqb_result_free(C.byref(res))
            _raise(st)
        out = self._collect(res, m, n, output)
        if st == 4:
            raise ToleranceNotReached(
                f"tolerance not reached after {out.blocks} blocks; residual "
                f"{np.sqrt(max(out.residual_sq, 0.0)):.6g}", out)
        if st == 3:
            raise BlockDegenerate(N.lib().fqb_last_error().decode(errors="replace"), out.blocks,
                                  out.residual_sq, out.norm_a_sq)
        return out

    def _make_source(self, source):
        if source is None:
            return N.SOURCE_FN(), [], None
        err: list = []
        keep: list = []

        def cb(_user, n, b, bid, out):
            try:
                blk = source.next(n, b, bid) if isinstance(source, BlockSource) else source(n, b, bid)
                keep.clear()
                c = N.BlockC()
                c.is_dense = int(blk.is_dense)
                c.rows, c.cols = int(blk.rows), int(blk.cols)
                c.centered = int(blk.centered)
                c.p = float(blk.p)
                c.std_scale = float(blk.std_scale)
                if blk.is_dense:
                    d = np.asfortranarray(blk.dense, dtype=np.float64)
                    keep.append(d)
                    c.dense = d.ctypes.data
                else:
                    cp = np.ascontiguousarray(blk.col_ptr, dtype=np.int32)
                    ri = np.ascontiguousarray(blk.row_idx, dtype=np.int32)
                    va = np.ascontiguousarray(blk.values, dtype=np.float64)
                    if ri.size == 0:
                        ri, va = np.zeros(1, np.int32), np.zeros(1)
                    keep.extend([cp, ri, va])
                    c.col_ptr, c.row_idx, c.values = cp.ctypes.data, ri.ctypes.data, va.ctypes.data
                    c.nnz = int(cp[-1])
                out[0] = c
                return 0
            except Exception as e:  # noqa: BLE001 - surfaced as CallbackError
                err.append(e)
                return 1

        fn = N.SOURCE_FN(cb)
        return fn, err, (fn, keep)

    def _collect(self, res: N.ResultC, m: int, n: int, output: str) -> QBResult:
        l = res.rank
        q = bt = None
        try:
            if l > 0 and output == "device" and res.q:
                import torch
                qb = _DeviceBuffer(res.q, m, l, res.ldq)
                bb = _DeviceBuffer(res.bt, n, l, res.ldbt)
                res.q = None
                res.bt = None
                with torch.cuda.device(self.device):
                    q = torch.as_tensor(qb, device=f"cuda:{self.device}").t()
                    bt = torch.as_tensor(bb, device=f"cuda:{self.device}").t()
            elif l > 0 and output == "host" and res.q:
                # zero-copy: the arrays own the library's pinned buffers
                q = _host_array(res.q, m, l)
                bt = _host_array(res.bt, n, l)
                res.q = None
                res.bt = None
            br = (np.ctypeslib.as_array(res.block_residuals, (res.blocks,)).copy()
                  if res.blocks and res.block_residuals else np.zeros(0))
            ids = (np.ctypeslib.as_array(res.block_ids, (res.n_ids,)).tolist()
                   if res.n_ids and res.block_ids else [])
            out = QBResult(q, bt, l, res.blocks, bool(res.converged), res.residual_sq, res.norm_a_sq,
                           br, [int(i) for i in ids], res.resolved_block, res.resolved_max_iters,
                           res.resolved_p, res.elapsed_ms, res.gpu_launches)
            if res.sigma:
                r = res.svd_rank
                out.sigma = np.ctypeslib.as_array(res.sigma, (max(r, 1),))[:r].copy()
                out.v_flagged = np.frombuffer(C.string_at(res.v_flagged, r), dtype=np.int8).astype(bool)
                out.svd_residual_sq = res.svd_residual_sq
                if r > 0 and res.u and output == "device":
                    import torch
                    ub = _DeviceBuffer(res.u, m, r, res.ldu)
                    vb = _DeviceBuffer(res.v, n, r, res.ldv)
                    res.u = None
                    res.v = None
                    with torch.cuda.device(self.device):
                        out.u = torch.as_tensor(ub, device=f"cuda:{self.device}").t()
                        out.v = torch.as_tensor(vb, device=f"cuda:{self.device}").t()
                elif r > 0 and res.u and output == "host":
                    out.u = _host_array(res.u, m, r)
                    out.v = _host_array(res.v, n, r)
                    res.u = None
                    res.v = None
            return out
        finally:
            self._lib.fqb_result_free(C.byref(res))

    # ---- building blocks ----------------------------------------------------
    def philox_u32(self, seed: int, block_id: int, column: int, count: int) -> np.ndarray:
        out = np.zeros(count, dtype=np.uint32)
        st = self._lib.fqb_philox_u32(self._h, seed, block_id, column, count, out.ctypes.data)
        if st:
            _raise(st, "fqb_philox_u32")
        return out

    def gen_sketch(self, spec: SketchSpec, n: int, l: int, block_id: int) -> SketchBlock:
        s = N.SketchHostC()
        cs = N.SketchSpecC(int(spec.kind), float(spec.p), int(spec.seed) & (2**64 - 1), int(spec.zeta))
        st = self._lib.fqb_gen_sketch(self._h, C.byref(cs), n, l, block_id, C.byref(s))
        if st:
            _raise(st, "fqb_gen_sketch")
        try:
            if s.is_dense:
                d = np.ctypeslib.as_array(s.dense, (n * l,)).reshape((n, l), order="F").copy()
                return SketchBlock(True, n, l, dense=d, p=s.p)
            nnz = int(s.nnz)
            cp = np.ctypeslib.as_array(s.col_ptr, (l + 1,)).copy()
            ri = np.ctypeslib.as_array(s.row_idx, (max(nnz, 1),))[:nnz].copy()
            va = np.ctypeslib.as_array(s.values, (max(nnz, 1),))[:nnz].copy()
            return SketchBlock(False, n, l, col_ptr=cp, row_idx=ri, values=va,
                               centered=bool(s.centered), p=s.p, std_scale=s.std_scale)
        finally:
            self._lib.fqb_sketch_free(C.byref(s))

    def gemm(self, trans_a: bool, m, n, k, alpha, a_ptr, lda, b_ptr, ldb, beta, c_ptr, ldc):
        st = self._lib.fqb_gemm(self._h, int(trans_a), m, n, k, alpha, a_ptr, lda, b_ptr, ldb, beta,
                                c_ptr, ldc)
        if st:
            _raise(st, "fqb_gemm")

    def gemm_emulated(self, trans_a: bool, m, n, k, alpha, a_ptr, lda, b_ptr, ldb, beta, c_ptr, ldc):
        """FP64 GEMM on the INT8 tensor cores (Ozaki slicing); n > 64 runs in chunks of <= 64 columns."""
        st = self._lib.fqb_gemm_emulated(self._h, int(trans_a), m, n, k, alpha, a_ptr, lda, b_ptr, ldb, beta,
                                         c_ptr, ldc)
        if st:
            _raise(st, "fqb_gemm_emulated")

    def relative_error(self, a, res: "QBResult") -> float:
        """rsvd::relative_error (experiment.cpp:317-342): ||A - U diag(sigma) V'||_F / ||A||_F on the
        device, one pass over A.  Uses the ApproxSvd factors when res has them, else Q and B."""
        ptr, m, n, lda, on_dev, keep, f32 = _as_colmajor(a)
        if f32:
            raise InvalidArgument("relative_error takes a float64 A")
        if res.sigma is not None and res.u is not None:
            fu, fv, sig = res.u, res.v, np.ascontiguousarray(res.sigma, dtype=np.float64)
        else:
            fu, fv, sig = res.q, res.bt, None
        r = 0 if fu is None else int(fu.shape[1])
        keep_f = []

        def fptr(x, rows):
            if x is None:
                return None, rows, False
            if _is_torch(x):
                xc = x if x.stride(0) == 1 else x.t().contiguous().t()
                keep_f.append(xc)
                return xc.data_ptr(), (xc.stride(1) if xc.shape[1] > 1 else rows), xc.is_cuda
            xa = np.asfortranarray(x, dtype=np.float64)
            keep_f.append(xa)
            return xa.ctypes.data, rows, False
        up, ldu, udev = fptr(fu, m)
        vp, ldv, vdev = fptr(fv, n)
        if r > 0 and udev != vdev:
            raise InvalidArgument("U and V must both be on the host or both on the device")
        out = C.c_double()
        st = self._lib.fqb_relative_error(self._h, ptr, m, n, lda, int(on_dev), up, max(ldu, 1),
                                          None if sig is None else sig.ctypes.data, vp, max(ldv, 1), r,
                                          int(bool(udev)), C.byref(out))
        del keep, keep_f
        if st:
            _raise(st, "fqb_relative_error")
        return out.value

    def set_fp32_slices(self, slices: int) -> None:
        """FP32 inputs: 8 slices per operand (FP64-class A passes, default), 4 or 3 (FP32-class,
        about twice as fast; fqb_set_fp32_slices)."""
        st = self._lib.fqb_set_fp32_slices(self._h, int(slices))
        if st:
            _raise(st, "fqb_set_fp32_slices")

    def sym_eig(self, a):
        """Symmetric eigendecomposition on the device (fqb_sym_eig, the SVD assembly's solver):
        a torch float64 n x n (CUDA) -> (w ascending, V) as torch tensors, and whether the
        small-l solver (rather than cuSOLVER) produced them."""
        import torch
        n = int(a.shape[0])
        ac = a.t().contiguous().t() if a.stride(0) != 1 else a
        w = torch.empty(n, dtype=torch.float64, device=a.device)
        v = torch.empty((n, n), dtype=torch.float64, device=a.device).t()
        used = C.c_int(0)
        st = self._lib.fqb_sym_eig(self._h, ac.data_ptr(), n, max(n, 1) if n <= 1 else ac.stride(1), w.data_ptr(),
                                   v.data_ptr(), max(n, 1), C.byref(used))
        if st:
            _raise(st, "fqb_sym_eig")
        return w, v, bool(used.value)

    def gram(self, y, out=None, sync: bool = True):
        """S = y' y (fqb_gram) for a tall column-major torch float64 y (CUDA) -> torch b x b."""
        import torch
        k, b = int(y.shape[0]), int(y.shape[1])
        ldy = y.stride(1) if (y.stride(0) == 1 and b > 1) else max(k, 1)
        if y.stride(0) != 1:
            raise InvalidArgument("gram: y must be column-major")
        s = out if out is not None else torch.empty((b, b), dtype=torch.float64, device=y.device).t()
        st = self._lib.fqb_gram(self._h, y.data_ptr(), k, b, ldy, s.data_ptr(), s.stride(1) if b > 1 else 1)
        if st:
            _raise(st, "fqb_gram")
        if sync:
            torch.cuda.synchronize(y.device)
        return s

    def mul_upper(self, y, r, sync: bool = True):
        """Z = y r with r upper triangular (fqb_mul_upper; r's strictly lower part is not read)."""
        import torch
        m, b = int(y.shape[0]), int(y.shape[1])
        if y.stride(0) != 1 or r.stride(0) != 1:
            raise InvalidArgument("mul_upper: column-major operands")
        z = torch.empty((b, m), dtype=torch.float64, device=y.device).t()
        st = self._lib.fqb_mul_upper(self._h, y.data_ptr(), m, b, y.stride(1) if b > 1 else max(m, 1), r.data_ptr(),
                                     r.stride(1) if b > 1 else 1, z.data_ptr(), max(m, 1))
        if st:
            _raise(st, "fqb_mul_upper")
        if sync:
            torch.cuda.synchronize(y.device)
        return z

    def chol_factor(self, z, pivot_tol: float = 1e-12, diag_ref: float = 0.0):
        """rsvd::chol_factor on the device (fqb_chol_factor): a symmetric torch float64 n x n
        (CUDA) -> (R = L', R^-1, rank_deficient) -- rank_deficient (R = R^-1 = I) when a pivot
        falls to pivot_tol * max_diag, the reference's RankDeficient."""
        import torch
        n = int(z.shape[0])
        zc = z.t().contiguous().t() if z.stride(0) != 1 else z
        r = torch.empty((n, n), dtype=torch.float64, device=z.device).t()
        ri = torch.empty((n, n), dtype=torch.float64, device=z.device).t()
        bad = C.c_int(0)
        st = self._lib.fqb_chol_factor(self._h, zc.data_ptr(), n, max(n, 1) if n <= 1 else zc.stride(1),
                                       float(pivot_tol), float(diag_ref), r.data_ptr(), max(n, 1), ri.data_ptr(),
                                       max(n, 1), C.byref(bad))
        if st:
            _raise(st, "fqb_chol_factor")
        return r, ri, bool(bad.value)

    # ---- test matrices on the device (reference synthetic.cpp) -------------------
    def random_orthonormal(self, n: int, r: int, seed: int, stream: int = 0xFA000001):
        """rsvd::random_orthonormal on the device -> torch float64 n x r (column-major)."""
        import torch
        q = torch.empty((r, n), dtype=torch.float64, device=f"cuda:{self.device}").t()
        st = self._lib.fqb_random_orthonormal(self._h, n, r, seed, stream, q.data_ptr(), max(n, 1))
        if st:
            _raise(st, "fqb_random_orthonormal")
        return q

    def gen_synthetic(self, kind: int, n: int, seed: int, d: int = 1):
        """rsvd::gen_synthetic on the device (kind 0 slow, 1 fast, 2 block-V) -> (A torch n x n, rank)."""
        import torch
        a = torch.empty((n, n), dtype=torch.float64, device=f"cuda:{self.device}").t()
        r = C.c_int()
        st = self._lib.fqb_gen_synthetic(self._h, int(kind), n, d, seed, a.data_ptr(), max(n, 1), C.byref(r))
        if st:
            _raise(st, "fqb_gen_synthetic")
        return a, r.value

    def gen_lowrank(self, m: int, n: int, sigma, seed: int, noise: float = 0.0):
        """A = U diag(sigma) V' + noise N(0,1)/sqrt(n) on the device (BASELINE configs 2-5)."""
        import torch
        sig = np.ascontiguousarray(np.asarray(sigma, dtype=np.float64))
        a = torch.empty((n, m), dtype=torch.float64, device=f"cuda:{self.device}").t()
        st = self._lib.fqb_gen_lowrank(self._h, m, n, len(sig), sig.ctypes.data, seed, float(noise), a.data_ptr(),
                                       max(m, 1))
        if st:
            _raise(st, "fqb_gen_lowrank")
        return a

    def gen_lowrank_det(self, m: int, n: int, sigma, seed: int, noise_scale: float = 0.0, row0: int = 0,
                        rows: int | None = None):
        """Rows [row0, row0 + rows) of the deterministic A = X diag(sigma) Y' + noise_scale G
        (fqb_gen_lowrank_det; bit-equal to the host twin oracle/detgen.c) -> torch rows x n."""
        import torch
        rows = m - row0 if rows is None else rows
        sig = np.ascontiguousarray(np.asarray(sigma, dtype=np.float64))
        a = torch.empty((n, rows), dtype=torch.float64, device=f"cuda:{self.device}").t()
        st = self._lib.fqb_gen_lowrank_det(self._h, m, n, len(sig), sig.ctypes.data, seed, float(noise_scale),
                                           row0, rows, a.data_ptr(), max(rows, 1))
        if st:
            _raise(st, "fqb_gen_lowrank_det")
        return a

    def checksum(self, a, row0: int = 0, m_total: int | None = None) -> int:
        """fqb_checksum of a device column-major torch matrix (a row shard starting at row0)."""
        rows, cols = a.shape
        out = C.c_uint64()
        st = self._lib.fqb_checksum(self._h, a.data_ptr(), rows, cols, max(a.stride(1), rows, 1), row0,
                                    rows + row0 if m_total is None else m_total, C.byref(out))
        if st:
            _raise(st, "fqb_checksum")
        return out.value

    def slice_operand(self, a_ptr, m, n, lda) -> "SlicedOperand":
        """Cut A (m x n, device, column-major) once into Ozaki slices (fqb_slice_operand)."""
        out = C.c_void_p()
        st = self._lib.fqb_slice_operand(self._h, a_ptr, m, n, lda, C.byref(out))
        if st:
            _raise(st, "fqb_slice_operand")
        return SlicedOperand(self, out, m, n)

    def sparse_dense_mul(self, a_ptr, m, n, lda, col_ptr_ptr, row_idx_ptr, values_ptr, l, z_ptr,
                         c_ptr, ldc):
        st = self._lib.fqb_sparse_dense_mul(self._h, a_ptr, m, n, lda, col_ptr_ptr, row_idx_ptr,
                                            values_ptr, l, z_ptr, c_ptr, ldc)
        if st:
            _raise(st, "fqb_sparse_dense_mul")

    def centering_column(self, a_ptr, m, n, lda, p, z_ptr):
        st = self._lib.fqb_centering_column(self._h, a_ptr, m, n, lda, p, z_ptr)
        if st:
            _raise(st, "fqb_centering_column")

    def frob_norm_sq(self, a_ptr, m, n, lda) -> float:
        out = C.c_double()
        st = self._lib.fqb_frob_norm_sq(self._h, a_ptr, m, n, lda, C.byref(out))
        if st:
            _raise(st, "fqb_frob_norm_sq")
        return out.value


_default_engines: dict = {}


def default_engine(device: int = 0) -> Engine:
    e = _default_engines.get(device)
    if e is None:
        e = _default_engines[device] = Engine(device)
    return e


def run_fixed_precision(a, cfg: FarpcaConfig, source: BlockSource | None = None,
                        output: str = "device", device: int = 0, svd: bool = True) -> QBResult:
    """rsvd::run_fixed_precision (driver.hpp:98-99) on the B200 engine: the QB factors
    plus, like the reference's ApproxSvd, U, sigma (ascending) and V."""
    return default_engine(device).run_fixed_precision(a, cfg, source, output, svd=svd)


def run_fixed_rank(a, rank: int, cfg: FarpcaConfig, source: BlockSource | None = None,
                   output: str = "device", device: int = 0, svd: bool = True) -> QBResult:
    """rsvd::run_fixed_rank (driver.hpp:101-103): QB of ceil(rank/b)*b columns and an
    ApproxSvd of exactly `rank` triplets (the overshoot dropped like drop_smallest)."""
    return default_engine(device).run_fixed_rank(a, rank, cfg, source, output, svd=svd)


def truncate_to_tolerance(res: QBResult, eps_rel: float, norm_a: float) -> QBResult:
    """rsvd::truncate_to_tolerance (driver.cpp:415-433) on an assembled result:
    drop the smallest triplets while the residual stays within (eps_rel*norm_a)^2."""
    import copy
    if eps_rel < 0.0 or norm_a < 0.0:
        raise ConfigError("truncate_to_tolerance: negative tolerance or norm")
    if res.sigma is None:
        raise InvalidArgument("truncate_to_tolerance needs an assembled SVD (svd=True)")
    target = eps_rel * norm_a
    budget = target * target * (1.0 + 1e-12)
    acc = res.svd_residual_sq
    drop = 0
    while drop < len(res.sigma):
        nxt = acc + res.sigma[drop] * res.sigma[drop]
        if nxt > budget:
            break
        acc = nxt
        drop += 1
    if drop == 0:
        return res
    out = copy.copy(res)
    out.sigma = res.sigma[drop:].copy()
    out.v_flagged = res.v_flagged[drop:].copy()
    out.u = res.u[:, drop:] if res.u is not None else None
    out.v = res.v[:, drop:] if res.v is not None else None
    out.svd_residual_sq = acc
    return out


def estimate_cost(m: float, n: float, l: float, power: int, block: int, p: float, kind: SketchKind):
    """rsvd::estimate_cost (driver.cpp:435-447): multiply-add counts of the dense
    (Gaussian) loop and the accelerated (sparse) loop, and their ratio."""
    if m < 1 or n < 1 or l < 1 or block < 1 or power < 0:
        raise ConfigError("estimate_cost: arguments must be positive")
    pw, b = float(power), float(block)
    common = 1.5 * (m + n) * l * l + pw * (2.0 * m * n * l + n * l * l + 2.0 * n * l * b)
    dense = 2.0 * m * n * l + common
    accel = dense
    if SketchKind(kind) != SketchKind.Gaussian:
        accel = m * n * l + m * n * l * p + m * np.sqrt(n * l) + common
    return dense, accel, accel / dense


def gen_sketch(spec: SketchSpec, n: int, l: int, block_id: int, device: int = 0) -> SketchBlock:
    """rsvd::gen_sketch (sketch.hpp:46), generated on the device."""
    return default_engine(device).gen_sketch(spec, n, l, block_id)


def relative_error(a, res: QBResult, device: int = 0) -> float:
    """rsvd::relative_error: exact ||A - U diag(sigma) V'||_F / ||A||_F (or ||A - Q B|| for a QB result)."""
    return default_engine(device).relative_error(a, res)
