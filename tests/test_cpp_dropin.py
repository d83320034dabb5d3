"""The C++ drop-in header (include/farqb/rsvd_b200.hpp) compiles against the C-ABI
and behaves like the reference API: CPU checks here, a real QB run under -m gpu."""
import os
import shutil
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2506_03859_b200", "lib")


def _build(tmp_path):
    cxx = shutil.which("g++")
    if not cxx:
        pytest.skip("no g++")
    exe = str(tmp_path / "drop_in")
    subprocess.run([cxx, "-std=c++17", "-O2", "-Wall", "-Wextra", "-I" + os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "drop_in.cpp"), "-L" + LIBDIR, "-lfarqb",
                    "-Wl,-rpath," + LIBDIR, "-o", exe], check=True)
    return exe


def test_dropin_compiles_and_runs_without_gpu(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe, "cpu"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASS" in r.stdout


@pytest.mark.gpu
def test_dropin_qb_on_gpu(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe, "gpu"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASS" in r.stdout


# ---- link-level drop-in: an unmodified reference-API caller relinked on librsvd_b200.so ----

REF_DIR = os.path.join(ROOT, "oracle", "_ref")
CALLER_REF = os.path.join(REF_DIR, "ref_caller_ref")
CALLER_B200 = os.path.join(REF_DIR, "ref_caller_b200")
DROPIN = os.path.join(LIBDIR, "librsvd_b200.so")


def _need_callers():
    if not (os.path.exists(CALLER_REF) and os.path.exists(CALLER_B200) and os.path.exists(DROPIN)):
        pytest.skip("reference-API callers not built (make -C oracle ref, needs the reference headers)")


def test_dropin_library_exports_the_reference_entry_points():
    """librsvd_b200.so defines rsvd::run_fixed_precision / run_fixed_rank with the exact
    mangled signatures of driver.hpp:98-103, and the relinked caller resolves them there
    (it is first in the caller's load order) while the rest of the API stays in the reference."""
    _need_callers()
    nm = subprocess.run(["nm", "-D", "-C", "--defined-only", DROPIN], capture_output=True, text=True).stdout
    assert "rsvd::run_fixed_precision(rsvd::DenseMatrix const&, rsvd::FarpcaConfig const&, rsvd::BlockSource*)" in nm
    assert "rsvd::run_fixed_rank(rsvd::DenseMatrix const&, int, rsvd::FarpcaConfig const&, rsvd::BlockSource*)" in nm
    assert "rsvd::gen_sketch" not in nm    # nothing else of the reference is replaced
    need = subprocess.run(["readelf", "-d", CALLER_B200], capture_output=True, text=True).stdout
    libs = [ln.split("[")[1].split("]")[0] for ln in need.splitlines() if "(NEEDED)" in ln]
    assert libs.index("librsvd_b200.so") < libs.index("librsvd_ref.so")
    ref_need = subprocess.run(["readelf", "-d", CALLER_REF], capture_output=True, text=True).stdout
    assert "librsvd_b200.so" not in ref_need


def _parse(out):
    cases = {}
    for line in out.splitlines():
        name, _, rest = line.partition(" ")
        kv = {}
        for tok in rest.split(" "):
            if "=" in tok:
                k, v = tok.split("=", 1)
                kv[k] = v
        if "what" in line:
            kv["what"] = line.split('what="', 1)[1].rsplit('"', 1)[0]
        cases[name] = kv
    return cases


def _nums(s):
    return np.array([float(x) for x in s.split(",")]) if s else np.zeros(0)


@pytest.mark.gpu
def test_dropin_reference_caller_matches_reference():
    """The same reference-API program, relinked on the B200 drop-in, prints the same
    factorizations as against the reference library: rank / blocks / converged / block
    ids / exception kinds and messages exact, residual within 1e-10 ||A||^2, sigma (>= 1e-3
    sigma_max) within 1e-10 sigma_max, a U diag(sigma) V' probe within 1e-10 ||A||_F."""
    _need_callers()
    ref = subprocess.run([CALLER_REF], capture_output=True, text=True, timeout=600)
    gpu = subprocess.run([CALLER_B200], capture_output=True, text=True, timeout=600)
    assert ref.returncode == 0, ref.stderr
    assert gpu.returncode == 0, gpu.stderr
    r, g = _parse(ref.stdout), _parse(gpu.stdout)
    assert sorted(r) == sorted(g)
    for name in r:
        a, b = r[name], g[name]
        assert a["status"] == b["status"], name
        if "what" in a:
            assert a["what"] == b["what"], name
        if a["status"] == "BlockDegenerate":
            assert a["blocks"] == b["blocks"], name
            na = float(a["norm_a_sq"])
            assert abs(float(a["residual_sq"]) - float(b["residual_sq"])) <= 1e-10 * na, name
        if a["status"] != "ok":
            continue
        for k in ("rank", "blocks", "converged", "ids"):
            assert a.get(k) == b.get(k), (name, k, a.get(k), b.get(k))
        na = float(a["norm_a_sq"])
        assert abs(float(b["norm_a_sq"]) - na) <= 1e-12 * na, name
        assert abs(float(a["residual_sq"]) - float(b["residual_sq"])) <= 1e-10 * na, name
        sa, sb = _nums(a["sigma"]), _nums(b["sigma"])
        top = sa >= 1e-3 * sa[-1]
        assert np.max(np.abs(sa[top] - sb[top])) <= 1e-10 * sa[-1], name
        assert np.max(np.abs(_nums(a["probe"]) - _nums(b["probe"]))) <= 1e-10 * np.sqrt(na) * 1.3, name
