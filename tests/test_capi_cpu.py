"""CPU-side checks of the drop-in boundary: the C-ABI library loads, exports
every symbol include/farqb.h declares, and refuses to compute without a GPU."""
import ctypes
import os
import re

import pytest

from paper_2506_03859_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "farqb.h")).read()
    return sorted(set(re.findall(r"\b(fqb_[a-z0-9_]+)\s*\(", text)) - {"fqb_block_source_fn"})


def test_header_and_binding_agree():
    bound = {name for name, _, _ in _native.SIGNATURES}
    assert set(declared_symbols()) == bound


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_native.LIB_PATH)
    for name in declared_symbols():
        assert hasattr(lib, name), name


def test_abi_version_and_defaults():
    L = _native.lib()
    assert L.fqb_abi_version() == 3
    # driver.cpp:449-466 heuristics, same numbers as test_driver.cpp:384-401
    assert L.fqb_default_block(100, 100) == 20
    assert L.fqb_default_block(3000, 3000) == 30
    assert L.fqb_default_block(20000, 20000) == 50
    assert L.fqb_default_block(10, 10) == 10
    assert L.fqb_default_max_iters(400, 20) == 10
    assert L.fqb_default_max_iters(401, 20) == 11
    assert L.fqb_default_max_iters(39, 20) == 1
    assert L.fqb_default_density(3, 20000) == 1e-3
    assert L.fqb_default_density(3, 1000) == 0.01
    assert L.fqb_default_density(0, 1000) == 0.0
    assert L.fqb_status_name(4) == b"tolerance_not_reached"


def test_no_gpu_means_loud_failure():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_2506_03859_b200 as fqb
    with pytest.raises(fqb.CudaError):
        fqb.Engine(0)


def test_python_api_mirrors_reference_names():
    import paper_2506_03859_b200 as fqb
    for name in ("run_fixed_precision", "run_fixed_rank", "gen_sketch", "FarpcaConfig", "SketchSpec",
                 "SketchKind", "BlockSource", "SketchBlock", "ConfigError", "DimensionError",
                 "BlockDegenerate", "ToleranceNotReached", "ConvergenceFailure", "ShiftConvention",
                 "default_density", "default_block", "default_max_iters"):
        assert hasattr(fqb, name), name
    assert fqb.sketch_kind_from_name("sparsesign") == fqb.SketchKind.SparseSign
    assert fqb.sketch_kind_name(fqb.SketchKind.StdBernoulli) == "stdbernoulli"
    with pytest.raises(fqb.ConfigError):
        fqb.sketch_kind_from_name("uniform")
