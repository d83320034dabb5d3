#!/usr/bin/env python
"""farPCA time-to-epsilon benchmark (BASELINE.json metric) on B200.

Workload: BASELINE.json configs[3] ("C4"), the largest configuration that fits one
GPU: A = X diag(sigma) Y', 100000 x 20000 FP64 (16 GB), rank 2000, sigma_i =
10^(-3i/2000), X, Y = Q of QR of seeded N(0,1) (the deterministic generator
fqb_gen_lowrank_det, seed 42 -- bit-identical to its host twin oracle/detgen.c, so the
reference's golden run tests/golden/c4.json is on this exact matrix); sparse-Gaussian
Omega with zeta = 8 nonzeros per column (seed 7), b = 100, P = 2, eps = 1e-3 relative.

One step = one full run_fixed_precision to eps (20 blocks, rank 2000) through the
engine -- the blocked QB loop plus the assembly of U, sigma, V, exactly what the
reference's run_fixed_precision returns -- with A resident in HBM (16 GB >> the 126 MB
L2, so no flush is needed between steps).  `e2e` repeats the step through the public
API with A in pinned host memory (the 16 GB H2D inside the timed region) and Q, B', U,
V returned to the host.  `roofline` times the dominant kernel live (k_ozaki on the
paired column chunks, W = A'Y at the C4 shape).  `cpu_baseline` / `--impl reference`
time the unmodified reference (oracle/_ref, single-threaded like the library) on a
bounded row sample of the same matrix and extrapolate (see cpu_sample()).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

--gpus N > 1 without torchrun re-launches itself under torch.distributed.run; every
rank makes only its own row shard of A (the generator's factor Grams run over all
rows, so the shards are bit-equal to rows of the whole) and the engine all-reduces
over NCCL (strong scaling: one problem, rows sharded).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

M, N = 100000, 20000
RANK_SIG = 2000
BLOCK, POWER, EPS, ZETA = 100, 2, 1e-3, 8
SEED_A, SEED_OMEGA = 42, 7
KIND_SPARSE_GAUSSIAN = 4
SAMPLE_ROWS = 2000          # reference arm, per step: the first rows of A, one block (~3.7 s)
CPU_BASELINE_ROWS = 6000    # our arm's cpu_baseline leg: one sample of ~11 s of CPU work
WORKLOAD = ("C4: A = X diag(10^(-3i/2000)) Y', 100000x20000 FP64, rank 2000; sparse Gaussian Omega "
            "zeta=8; b=100, P=2, eps=1e-3 relative")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--workload", default="c4", choices=["c4", "c2"],
                    help="c4: the headline (configs[3]); c2: configs[1], a secondary line (one GPU)")
    return ap.parse_args()


def sigma():
    import numpy as np
    return 10.0 ** (-3.0 * np.arange(1, RANK_SIG + 1, dtype=np.float64) / RANK_SIG)


def peaks():
    """Roofline denominators: MEASURED_PEAKS.json (driver-written) for HBM; the FP64
    DMMA peak measured by this repo (profiles/fp64_peak_r01.txt) for context."""
    out = {"hbm_gbs": None, "source": "MEASURED_PEAKS.json", "fp64_tflops": 37.1,
           "fp64_source": "profiles/fp64_peak_r01.txt (DMMA microbenchmark; no FP64 entry in MEASURED_PEAKS.json)",
           "bf16_tflops": None}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            mp = json.load(f)
        out["hbm_gbs"] = float(mp["hbm_gbs"])
        out["bf16_tflops"] = float(mp["bf16_tflops"])
        if mp.get("bf16_tflops_sustained"):
            out["bf16_tflops_sustained"] = float(mp["bf16_tflops_sustained"])
    except (OSError, ValueError, KeyError):
        out["hbm_gbs"] = 6650.0
        out["source"] = "fallback (B200_PROFILING.md: 6.65 TB/s)"
    return out


def ozaki_int8_ops(rows_out: int, k: int, b: int) -> float:
    """INT8 tensor-core operations one k_ozaki<*,7,*,50|56> launch executes (2 per MAC): per
    128-row output tile, per 64-byte k-block and per column chunk the schedule runs MMAs
    of total N = 1744 for chunks of <= 50 columns (50-row Z spacing, 10 MMAs per 32-byte
    k-step) or 1936 for chunks of <= 56 (ozaki.cu).  Equals ncu's
    sm__ops_path_tensor_op_utcimma_src_int8_sparsity_off.sum (profiles/R3_ncu_ozaki_c4_s50_tn.txt)."""
    tiles = -(-rows_out // 128)
    kblocks = -(-k // 64)
    chunks = -(-b // 56)
    width = -(-b // chunks)
    n_rows = 1744 if width <= 50 else 1936
    return 2.0 * tiles * kblocks * chunks * n_rows * 128 * 64


def bench_config(world: int) -> dict:
    """The workload description -- identical in both arms."""
    return {"workload": WORKLOAD, "m": M, "n": N, "rank_signal": RANK_SIG, "sigma": "10^(-3i/2000), i=1..2000",
            "sketch": "sparse gaussian", "zeta": ZETA, "block": BLOCK, "power": POWER, "eps": EPS,
            "relative": True, "seed_a": SEED_A, "seed_omega": SEED_OMEGA,
            "generator": "fqb_gen_lowrank_det == oracle/detgen.c (bit-identical)",
            "step": "run_fixed_precision to eps + assemble_svd (U, sigma, V)",
            "l2": "A (16 GB) exceeds the 126 MB L2; no flush needed",
            "parallelism": f"rows of A sharded over {world} GPUs, NCCL all-reduce" if world > 1 else "single GPU"}


def config():
    from paper_2506_03859_b200 import FarpcaConfig, SketchKind, SketchSpec
    return FarpcaConfig(eps=EPS, power=POWER, block=BLOCK,
                        sketch=SketchSpec(SketchKind.SparseGaussian, 0.0, SEED_OMEGA, zeta=ZETA), relative=True)


def make_matrix(eng, row0=0, rows=None):
    """Rows [row0, row0 + rows) of C4's A on the device (fqb_gen_lowrank_det)."""
    return eng.gen_lowrank_det(M, N, sigma(), SEED_A, 0.0, row0, M - row0 if rows is None else rows)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, val in zip(names, parts[3:7]):
                if val.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def ozaki_roofline(eng, a, stream, pk):
    """Live per-launch timing of the dominant kernel: k_ozaki on the paired column chunks
    (b = 100 -> two chunks of 50 on multicast CTA pairs, + its stream-K fixup), W = A'Y at
    the C4 shape, on A and Y sliced beforehand (fqb_slice_operand / fqb_sliced_gemm_again),
    CUDA events on the launching stream.  Algorithmic bytes = SURVEY 8(d)'s dense A'Y figure
    8(mn + mb + nb) (FP64 A read once, Y read, W written); the kernel actually streams the
    7-byte slices of A (7mn), reported beside it.  The same A pass as the loop runs it (with
    the per-pass slicing of Y, k_slice_z) and the NN pass Y = A G are timed too."""
    import torch
    m, n = a.shape
    b = BLOCK
    y = torch.randn(b, m, dtype=torch.float64, device=a.device).t()
    w = torch.empty(b, n, dtype=torch.float64, device=a.device).t()
    g = torch.randn(b, n, dtype=torch.float64, device=a.device).t()
    yn = torch.empty(b, m, dtype=torch.float64, device=a.device).t()
    from paper_2506_03859_b200 import _native
    nsl = int(_native.lib().fqb_fp64_slices())
    out = {"nsl": nsl}
    sl = eng.slice_operand(a.data_ptr(), m, n, a.stride(1))
    reps = 6
    try:
        for name, trans, outp, bp in (("tn", True, w, y), ("nn", False, yn, g)):
            rows, k = (n, m) if trans else (m, n)
            for kind in ("pass", "kernel"):
                sl.gemm(trans, b, 1.0, bp.data_ptr(), bp.stride(1), 0.0, outp.data_ptr(), outp.stride(1))

                def call():
                    if kind == "pass":
                        sl.gemm(trans, b, 1.0, bp.data_ptr(), bp.stride(1), 0.0, outp.data_ptr(), outp.stride(1))
                    else:
                        sl.gemm_again(1.0, 0.0, outp.data_ptr(), outp.stride(1))
                for _ in range(2):
                    call()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                with torch.cuda.stream(stream):
                    e0.record()
                    for _ in range(reps):
                        call()
                    e1.record()
                e1.synchronize()
                ms = e0.elapsed_time(e1) / reps
                alg = 8.0 * (m * n + k * b + rows * b)
                out[f"{name}_{kind}"] = {"ms": ms, "gbs": alg / ms / 1e6, "bytes": alg,
                                         "slice_gbs": (nsl * m * n + 8.0 * (k * b + rows * b)) / ms / 1e6,
                                         "fp64_tflops_equiv": 2.0 * m * n * b / ms / 1e9}
    finally:
        sl.free()
    return out


def tensor_view(ms: float, pk: dict) -> dict:
    """The same launch against the INT8 tensor pipe, the unit that actually bounds it
    (DESIGN.md 4a): executed INT8 ops / launch time, against the dense INT8 rate (2x bf16
    per clock on B200: 4.5 POPS nominal, and 2x the MEASURED bf16 cuBLAS rate, i.e. the
    same power-capped clocks)."""
    ops = ozaki_int8_ops(N, M, BLOCK)
    tops = ops / ms / 1e9
    meas = 2.0 * pk["bf16_tflops"] if pk.get("bf16_tflops") else None
    sus = 2.0 * pk["bf16_tflops_sustained"] if pk.get("bf16_tflops_sustained") else None
    return {"int8_ops_per_launch": ops, "achieved_tops": tops, "peak_nominal_tops": 4500.0,
            "frac_nominal": tops / 4500.0, "peak_measured_equiv_tops": meas,
            "frac_measured_equiv": (tops / meas) if meas else None,
            "peak_measured_sustained_equiv_tops": sus,
            "frac_measured_sustained_equiv": (tops / sus) if sus else None,
            "note": "peak_measured_equiv = 2 x MEASURED_PEAKS bf16_tflops (burst), _sustained_ = 2 x "
                    "bf16_tflops_sustained (seconds-long, power-capped: the regime of the timed step); "
                    "no INT8 entry in MEASURED_PEAKS.json"}


def sketch_roofline(eng, dev, pk):
    """Sparse-sign sketch Y = A*Omega at BASELINE config 3's shape (A 20000 x 20000 FP64,
    b = 64, zeta = 8): HBM GB/s of the gather SpMM.  32 different Omega blocks, each writing
    its own Y (32 x 10 MB > L2), so neither the column reads nor the Y writes of one launch
    are served from L2 by the previous one."""
    import numpy as np
    import torch
    from paper_2506_03859_b200 import SketchKind, SketchSpec
    m = n = 20000
    b, zeta, nblk = 64, 8, 32
    a = torch.randn(n, m, dtype=torch.float64, device=dev).t()      # m x n column-major
    spec = SketchSpec(SketchKind.SparseSign, 0.0, 7, zeta=zeta)
    blocks, alg_bytes = [], []
    for j in range(nblk):
        s = eng.gen_sketch(spec, n, b, j)
        u = len(np.unique(s.row_idx))
        blocks.append((torch.from_numpy(s.col_ptr.astype(np.int32)).to(dev),
                       torch.from_numpy(s.row_idx.astype(np.int32)).to(dev),
                       torch.from_numpy(s.values).to(dev),
                       torch.empty(b, m, dtype=torch.float64, device=dev).t()))
        alg_bytes.append(8 * m * (u + b) + 12 * s.nnz + 4 * (b + 1))
    stream = torch.cuda.Stream(device=dev)
    eng.set_stream(stream.cuda_stream)

    def launch(j):
        cp, ri, va, y = blocks[j]
        eng.sparse_dense_mul(a.data_ptr(), m, n, m, cp.data_ptr(), ri.data_ptr(), va.data_ptr(), b, None,
                             y.data_ptr(), m)
    for j in range(nblk):
        launch(j)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 4
    e0.record(stream)
    for _ in range(reps):
        for j in range(nblk):
            launch(j)
    e1.record(stream)
    e1.synchronize()
    ms = e0.elapsed_time(e1) / (reps * nblk)
    gbs = (sum(alg_bytes) / nblk) / (ms * 1e-3) / 1e9
    del a, blocks
    torch.cuda.empty_cache()
    return {"kernel": "k_gather_spmm (sparse sign, zeta=8) Y = A*Omega, A 20000x20000, b=64, 32 distinct Y",
            "achieved": gbs, "peak": pk["hbm_gbs"], "unit": "GB/s", "frac": gbs / pk["hbm_gbs"],
            "launch_us": ms * 1e3, "bytes_per_launch": sum(alg_bytes) / nblk,
            "bytes_formula": "8*m*(u+b) + 12*nnz + 4*(b+1), u = distinct rows of the block"}


def load_traffic():
    for name in ("R4_traffic.json", "R3_traffic.json", "R2_traffic.json"):
        try:
            with open(os.path.join(ROOT, "profiles", name)) as f:
                return json.load(f)
        except (OSError, ValueError):
            continue
    return None


def host_info():
    cpu = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    cpu = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu": cpu, "nproc": os.cpu_count()}


def cpu_sample(a_rows, blocks_full):
    """The unmodified reference (oracle/_ref; else the C port) on a bounded sample of the
    workload: the first SAMPLE_ROWS rows of A (SAMPLE_ROWS x 20000), one block (max_iters
    = 1: the sparse sketch, 2P+1 = 5 dense passes, CholQR, B update), single-threaded like
    the library (kernels.hpp:5-8).  Extrapolated to time-to-eps on the whole matrix as
    t_sample * (M / SAMPLE_ROWS) * blocks_full: every pass over A scales with its rows and
    the run repeats the block blocks_full times.  This leaves out the costs that grow with
    the accumulated rank (deflation, re-orthogonalisation against l up to 2000, the l x l
    Jacobi of assemble_svd), so it UNDER-states the reference's time; the full C4 reference
    run, measured once on the build host, is in tests/golden/c4.json."""
    import numpy as np
    from oracle.oracle import REF_LIB, Oracle
    which = "reference" if os.path.exists(REF_LIB) else "port"
    orc = Oracle(which)
    a = np.asfortranarray(a_rows)

    def src(nn, bb, bid):
        return orc_port().gen_sketch(KIND_SPARSE_GAUSSIAN, 0.0, SEED_OMEGA, nn, bb, bid, zeta=ZETA)
    t0 = time.perf_counter()
    r = orc.run(a, eps=EPS, power=POWER, block=BLOCK, kind=KIND_SPARSE_GAUSSIAN, seed=SEED_OMEGA, zeta=ZETA,
                max_iters=1, relative=True, source=src)
    dt = time.perf_counter() - t0
    scale = (M / a.shape[0]) * blocks_full
    return dt, dt * scale, which, r


_PORT = None


def orc_port():
    global _PORT
    if _PORT is None:
        from oracle.oracle import Oracle
        _PORT = Oracle("port")
    return _PORT


def full_reference_record():
    try:
        with open(os.path.join(ROOT, "tests", "golden", "c4.json")) as f:
            g = json.load(f)
        return {"seconds": g["reference_seconds"], "host": g["host"], "rank": g["rank"], "blocks": g["blocks"],
                "source": "tests/golden/c4.json (one full reference run on the build host, 1 core)"}
    except (OSError, ValueError, KeyError):
        return None


def maybe_spawn(args):
    """--gpus N > 1 outside torchrun: re-launch under torch.distributed.run on 127.0.0.1."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return False
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def run_ours(args):
    import numpy as np
    import torch

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    pk = peaks()

    import paper_2506_03859_b200 as fqb
    from paper_2506_03859_b200.dist import partition_rows
    eng = fqb.Engine(local)
    stream = torch.cuda.Stream(device=dev)
    eng.set_stream(stream.cuda_stream)
    r0, r1 = partition_rows(M, world, rank) if world > 1 else (0, M)
    a = make_matrix(eng, r0, r1 - r0)           # this rank's row shard only
    if world > 1:
        eng.attach_comm()
    torch.cuda.synchronize()
    cfg = config()

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    clk = ClockSampler(local).__enter__()
    t_wait = time.time()
    while not clk.lines and time.time() - t_wait < 10.0:   # NVML start-up must not overlap the timing
        time.sleep(0.05)
    for _ in range(max(args.warmup, 0)):
        r = eng.run_fixed_precision(a, cfg, output="device", svd=True)
        del r
    barrier()
    eng.set_pass_timing(True)    # CUDA events around every A-pass k_ozaki launch inside the timed steps
    launches0 = eng.launch_count
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    step_ms = []
    with torch.cuda.stream(stream):
        e0.record()
    last = None
    for _ in range(args.steps):
        # like rsvd::run_fixed_precision: QB loop + assemble_svd (U, sigma, V), all on the device.
        # The previous step's factors are released first (as a caller that consumed them would).
        last = None
        r = eng.run_fixed_precision(a, cfg, output="device", svd=True)
        step_ms.append(r.elapsed_ms)
        last, r = r, None
    with torch.cuda.stream(stream):
        e1.record()
    e1.synchronize()
    barrier()
    launches = eng.launch_count - launches0
    live_ms, live_n, live_bytes = eng.pass_timing()
    eng.set_pass_timing(False)
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = t.item()
    result = {"rank": last.rank, "blocks": last.blocks, "converged": bool(last.converged),
              "rel_error_indicator": float(np.sqrt(max(last.residual_sq, 0) / last.norm_a_sq)),
              "step_device_ms": step_ms}
    last = None

    # ---- e2e: pinned host A (this rank's rows) -> public API -> Q, B', U, V on the host --
    m_loc = a.shape[0]
    a_host = torch.empty((N, m_loc), dtype=torch.float64, pin_memory=True)   # (n x m) row-major == A col-major
    a_host.copy_(a.t())
    a_host_cm = a_host.t()
    eng.run_fixed_precision(a_host_cm, cfg, output="host", svd=True)
    torch.cuda.synchronize()
    t_e2e = []
    r = None
    e2e_steps = max(1, args.steps)   # the same K as the device-timed steps
    for _ in range(e2e_steps):
        r = None   # the caller is done with the previous factors (their pinned blocks return to the pool)
        barrier()
        t0 = time.perf_counter()
        r = eng.run_fixed_precision(a_host_cm, cfg, output="host", svd=True)
        t_e2e.append(time.perf_counter() - t0)
    e2e_s = statistics.mean(t_e2e)
    clk.__exit__(None, None, None)
    h2d = m_loc * N * 8
    # Q, B' and U, V (m x l, n x l each), sigma, flags and the per-block trace
    d2h = 2 * (m_loc + N) * r.rank * 8 + 9 * r.rank + 8 * (r.blocks + 4)
    r = None
    del a_host, a_host_cm
    if world > 1:
        t = torch.tensor([e2e_s], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_s = t.item()

    roof = ozaki_roofline(eng, a, stream, pk)
    a_rows = a[:CPU_BASELINE_ROWS].cpu().numpy() if (rank == 0 and world == 1 and not args.no_cpu_baseline) else None
    del a
    torch.cuda.empty_cache()
    sketch = sketch_roofline(eng, dev, pk)
    dom = roof["tn_kernel"]   # the dominant kernel by itself (k_ozaki + its stream-K fixup)
    live_launch_ms = live_ms / max(live_n, 1)
    live_gbs = (live_bytes / max(live_n, 1)) / live_launch_ms / 1e6 if live_n else 0.0
    traffic = load_traffic()
    line = {
        "metric": "farPCA time-to-eps (s)",
        "value": ms / 1000.0,
        "unit": "s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": False,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic: C4's A from fqb_gen_lowrank_det (seed 42), bit-identical to oracle/detgen.c",
        "config": bench_config(world),
        "result": result,
        "e2e": {"value": e2e_s, "unit": "s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "steps": e2e_steps},
        "gpu_launches": launches,
        "roofline": {"bound": "hbm",
                     "kernel": "k_ozaki<true,7,2,50> (tcgen05 kind::i8 FP64 emulation, two 50-column chunks on "
                               "multicast CTA pairs) + k_ozaki_fixup: the A passes W = A'Y and Y = A G of the timed "
                               "steps",
                     "achieved": live_gbs, "peak": pk["hbm_gbs"], "unit": "GB/s",
                     "frac": live_gbs / pk["hbm_gbs"], "traffic": (traffic or {}).get("ozaki_c4_tn_bytes_per_launch"),
                     "traffic_source": (traffic or {}).get("source"),
                     "peak_source": pk["source"],
                     "timing": "live: CUDA events on the engine's stream around every A-pass k_ozaki launch (+ fixup) "
                               "inside the timed steps (fqb_set_pass_timing / fqb_pass_timing)",
                     "launches_timed": live_n, "launch_ms": live_launch_ms,
                     "bytes_per_launch": live_bytes / max(live_n, 1),
                     "bytes_formula": "8*(M*K + K*b + M*b) per launch (SURVEY 8(d): FP64 A read once, Y read, W "
                                      "written) = 8*(m*n + m*b + n*b) at C4",
                     "slice_bytes_per_launch": roof["nsl"] * M * N + 8.0 * (M * BLOCK + N * BLOCK),
                     "fp64_tflops_equiv": 2.0 * M * N * BLOCK / live_launch_ms / 1e9,
                     "fp64_peak_tflops": pk["fp64_tflops"],
                     "tensor_view": tensor_view(live_launch_ms, pk),
                     "isolated": {"what": "the same products outside the loop on the bench matrix, 6 back-to-back "
                                          "launches each (fqb_sliced_gemm / _again)",
                                  "tn_kernel_ms": dom["ms"], "nn_kernel_ms": roof["nn_kernel"]["ms"],
                                  "tn_pass_ms": roof["tn_pass"]["ms"], "nn_pass_ms": roof["nn_pass"]["ms"]}},
        "sketch_roofline": sketch,
        "clocks": clk.summary(),
    }
    if a_rows is not None:
        dt, est, which, rr = cpu_sample(a_rows, result["blocks"])
        line["cpu_baseline"] = {"value": est, "unit": "s", "cores": 1, "kind": which,
                                "sample": f"reference run_fixed_precision on rows [0,{CPU_BASELINE_ROWS}) of A, 1 block "
                                          f"(max_iters=1): {dt:.2f} s; x (m/{CPU_BASELINE_ROWS}) x {result['blocks']} "
                                          "blocks (excludes the rank-dependent costs, so a lower bound)",
                                "sample_seconds": dt, "host": host_info(),
                                "full_run_on_build_host": full_reference_record()}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def run_reference(args):
    """--impl reference: the reference's own CPU run_fixed_precision (oracle/_ref) on the
    bounded sample of cpu_sample(), each step one sample, value extrapolated to C4."""
    import numpy as np
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import ctypes as C
    from oracle.oracle import PORT_LIB
    lib = C.CDLL(PORT_LIB)
    lib.fqo_det_lowrank.argtypes = [C.c_int64, C.c_int64, C.c_int, C.c_void_p, C.c_uint64, C.c_double, C.c_int64,
                                    C.c_int64, C.c_void_p, C.c_int64]
    sig = sigma()
    a = np.empty((N, SAMPLE_ROWS), dtype=np.float64).T        # the same rows the ours arm samples, host-made
    st = lib.fqo_det_lowrank(M, N, len(sig), sig.ctypes.data, SEED_A, 0.0, 0, SAMPLE_ROWS, a.ctypes.data,
                             SAMPLE_ROWS)
    if st:
        print(json.dumps({"impl": "reference", "unavailable": f"fqo_det_lowrank failed ({st})"}))
        return
    full = full_reference_record()
    blocks_full = full["blocks"] if full else 20
    times, ests = [], []
    for i in range(max(args.warmup, 0) + args.steps):
        dt, est, which, r = cpu_sample(a, blocks_full)
        if i >= args.warmup:
            times.append(dt)
            ests.append(est)
    v = statistics.mean(ests)
    # n_gpus echoes the launch (--gpus N) so the line pairs with our arm's; the work runs on host cores
    line = {"metric": "farPCA time-to-eps (s)", "value": v, "unit": "s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": v * 1000,
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: the same A (oracle/detgen.c rows = fqb_gen_lowrank_det rows)", "impl": "reference",
            "config": bench_config(args.gpus),
            "cpu_baseline": {"value": v, "unit": "s", "cores": 1, "kind": which,
                             "sample": f"each step: reference run_fixed_precision on rows [0,{SAMPLE_ROWS}) of A, "
                                       f"1 block (mean {statistics.mean(times):.2f} s); value = x (m/{SAMPLE_ROWS}) x "
                                       f"{blocks_full} blocks (a lower bound: rank-dependent costs excluded)",
                             "sample_seconds": times, "host": host_info(), "full_run_on_build_host": full},
            "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---- secondary line: BASELINE configs[1] (C2), opt-in with --workload c2 ----------------
C2_N, C2_RANK, C2_BLOCK, C2_POWER, C2_EPS = 8000, 900, 50, 2, 1e-3
C2_WORKLOAD = ("C2: A = U diag(10^(-i/50)) V', 8000x8000 FP64 (fqb_gen_lowrank_det seed 42, 900 singular values "
               "kept: sigma_900 = 1e-18); StdBernoulli Omega p=1/2; b=50, P=2, eps=1e-3 relative")


def c2_sigma():
    import numpy as np
    return 10.0 ** (-np.arange(1, C2_RANK + 1, dtype=np.float64) / 50.0)


def c2_config_dict():
    return {"workload": C2_WORKLOAD, "m": C2_N, "n": C2_N, "block": C2_BLOCK, "power": C2_POWER, "eps": C2_EPS,
            "relative": True, "sketch": "stdbernoulli", "p": 0.5, "seed_a": SEED_A, "seed_omega": SEED_OMEGA,
            "step": "run_fixed_precision to eps + assemble_svd (U, sigma, V)",
            "l2": "A (512 MB) exceeds the 126 MB L2; no flush needed", "parallelism": "single GPU"}


def run_c2(args):
    """C2 on one GPU: device time with A resident, e2e from pinned host A with Q, B', U, V
    returned, and the unmodified reference (oracle/_ref, 1 core) timed on the whole run."""
    import numpy as np
    import torch
    import paper_2506_03859_b200 as fqb
    from paper_2506_03859_b200 import FarpcaConfig, SketchKind, SketchSpec
    if int(os.environ.get("RANK", "0")) != 0:
        return
    dev = torch.device("cuda:0")
    eng = fqb.Engine(0)
    stream = torch.cuda.Stream(device=dev)
    eng.set_stream(stream.cuda_stream)
    a = eng.gen_lowrank_det(C2_N, C2_N, c2_sigma(), SEED_A)
    cfg = FarpcaConfig(eps=C2_EPS, power=C2_POWER, block=C2_BLOCK,
                       sketch=SketchSpec(SketchKind.StdBernoulli, 0.5, SEED_OMEGA), relative=True)
    torch.cuda.synchronize()
    clk = ClockSampler(0).__enter__()
    t_wait = time.time()
    while not clk.lines and time.time() - t_wait < 10.0:
        time.sleep(0.05)
    for _ in range(max(args.warmup, 0)):
        eng.run_fixed_precision(a, cfg, output="device", svd=True)
    torch.cuda.synchronize()
    eng.set_pass_timing(True)
    launches0 = eng.launch_count
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record()
    last = None
    for _ in range(args.steps):
        last = None
        last = eng.run_fixed_precision(a, cfg, output="device", svd=True)
    with torch.cuda.stream(stream):
        e1.record()
    e1.synchronize()
    launches = eng.launch_count - launches0
    live_ms, live_n, _ = eng.pass_timing()
    eng.set_pass_timing(False)
    ms = e0.elapsed_time(e1) / args.steps
    rank_l, blocks = last.rank, last.blocks
    last = None
    a_host = torch.empty((C2_N, C2_N), dtype=torch.float64, pin_memory=True)
    a_host.copy_(a.t())
    a_host_cm = a_host.t()
    eng.run_fixed_precision(a_host_cm, cfg, output="host", svd=True)
    t_e2e, r = [], None
    for _ in range(max(1, args.steps)):
        r = None
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = eng.run_fixed_precision(a_host_cm, cfg, output="host", svd=True)
        t_e2e.append(time.perf_counter() - t0)
    clk.__exit__(None, None, None)
    d2h = 2 * (C2_N + C2_N) * r.rank * 8 + 9 * r.rank + 8 * (r.blocks + 4)
    r = None
    pk = peaks()
    launch_ms = live_ms / max(live_n, 1)
    bytes_launch = 8.0 * (C2_N * C2_N + 2 * C2_N * C2_BLOCK)
    ref = None
    if not args.no_cpu_baseline:
        ref = c2_reference_time(a.cpu().numpy())
    line = {"metric": "farPCA time-to-eps (s)", "value": ms / 1e3, "unit": "s", "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: C2's A from fqb_gen_lowrank_det (seed 42), bit-identical to oracle/detgen.c",
            "config": c2_config_dict(),
            "result": {"rank": rank_l, "blocks": blocks},
            "e2e": {"value": statistics.mean(t_e2e), "unit": "s", "h2d_bytes_per_step": C2_N * C2_N * 8,
                    "d2h_bytes_per_step": d2h, "steps": len(t_e2e)},
            "gpu_launches": int(launches),
            "roofline": {"bound": "hbm", "kernel": "k_ozaki (A passes, one 50-column chunk) + fixup, live",
                         "achieved": bytes_launch / (launch_ms * 1e-3) / 1e9, "peak": pk["hbm_gbs"],
                         "unit": "GB/s", "frac": bytes_launch / (launch_ms * 1e-3) / 1e9 / pk["hbm_gbs"],
                         "traffic": ((load_traffic() or {}).get("c2") or {}).get("bytes_per_launch"),
                         "traffic_source": ((load_traffic() or {}).get("c2") or {}).get("source"),
                         "launch_ms": launch_ms, "launches_timed": live_n,
                         "bytes_formula": "8*(m*n + m*b + n*b) per launch"},
            "clocks": clk.summary()}
    if ref:
        line["cpu_baseline"] = {"value": ref[0], "unit": "s", "cores": 1, "kind": ref[1],
                                "sample": "the whole C2 run (run_fixed_precision + assemble_svd), one core",
                                "host": host_info(), "rank": ref[2], "blocks": ref[3]}
    print(json.dumps(line), flush=True)


def c2_reference_time(a):
    """The unmodified reference's run_fixed_precision on the whole C2 matrix (one core)."""
    from oracle.oracle import REF_LIB, Oracle
    which = "reference" if os.path.exists(REF_LIB) else "port"
    orc = Oracle(which)
    t0 = time.perf_counter()
    r = orc.run(a, eps=C2_EPS, power=C2_POWER, block=C2_BLOCK, kind=2, p=0.5, seed=SEED_OMEGA, relative=True)
    return time.perf_counter() - t0, which, r.rank, r.blocks


def run_reference_c2(args):
    import numpy as np
    import ctypes as C
    if int(os.environ.get("RANK", "0")) != 0:
        return
    from oracle.oracle import PORT_LIB
    lib = C.CDLL(PORT_LIB)
    lib.fqo_det_lowrank.argtypes = [C.c_int64, C.c_int64, C.c_int, C.c_void_p, C.c_uint64, C.c_double, C.c_int64,
                                    C.c_int64, C.c_void_p, C.c_int64]
    sig = c2_sigma()
    a = np.empty((C2_N, C2_N), dtype=np.float64).T
    st = lib.fqo_det_lowrank(C2_N, C2_N, len(sig), sig.ctypes.data, SEED_A, 0.0, 0, C2_N, a.ctypes.data, C2_N)
    if st:
        print(json.dumps({"impl": "reference", "unavailable": f"fqo_det_lowrank failed ({st})"}))
        return
    ts = []
    for i in range(max(args.warmup, 0) + args.steps):
        dt, which, rk, bl = c2_reference_time(a)
        if i >= args.warmup:
            ts.append(dt)
    v = statistics.mean(ts)
    print(json.dumps({"metric": "farPCA time-to-eps (s)", "value": v, "unit": "s", "n_gpus": args.gpus,
                      "steps": args.steps, "warmup": args.warmup, "ms_per_step": v * 1e3, "higher_is_better": False,
                      "scaling": "strong", "vs_baseline": None, "dtype": "f64", "impl": "reference",
                      "data": "synthetic: the same A (oracle/detgen.c == fqb_gen_lowrank_det)",
                      "config": c2_config_dict(), "result": {"rank": rk, "blocks": bl},
                      "cpu_baseline": {"value": v, "unit": "s", "cores": 1, "kind": which,
                                       "sample": "each step the whole C2 run, one core", "sample_seconds": ts,
                                       "host": host_info()},
                      "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}),
          flush=True)


if __name__ == "__main__":
    a = parse()
    if a.workload == "c2":
        run_reference_c2(a) if a.impl == "reference" else run_c2(a)
    elif a.impl == "reference":
        run_reference(a)
    else:
        maybe_spawn(a)
        run_ours(a)
