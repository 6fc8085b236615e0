"""C-ABI checks that need no GPU: the library builds, loads, exports every declared symbol, its
descriptor layout matches the ctypes mirror, and argument validation returns the documented codes
before any device work (include/mrfnufft.h "Errors")."""
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mrfnufft.h")


@pytest.fixture(scope="module")
def binding():
    from paper_2310_05647_b200 import build
    build.build()
    from paper_2310_05647_b200 import binding as b
    return b


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mrf_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for required in ("mrf_plan_create", "mrf_forward", "mrf_adjoint", "mrf_normal", "mrf_dc_cg",
                     "mrf_plan_destroy", "mrf_status_string"):
        assert required in names


def test_library_exports_every_declared_symbol(binding):
    names = declared_functions()
    out = subprocess.run(["nm", "-D", "--defined-only", binding.LIB_PATH], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r"\bT (mrf_[a-z0-9_]+)\b", out))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    assert set(binding.EXPORTED) == set(names)


def test_library_is_sm100a(binding):
    out = subprocess.run(["cuobjdump", "--list-elf", binding.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_desc_layout_matches_ctypes(binding, tmp_path):
    prog = tmp_path / "layout.c"
    prog.write_text(
        '#include <stdio.h>\n#include <stddef.h>\n#include "mrfnufft.h"\n'
        "int main(void){printf(\"%zu %zu %zu %zu %zu %zu %zu\\n\", sizeof(mrf_plan_desc),"
        " offsetof(mrf_plan_desc, traj), offsetof(mrf_plan_desc, coils), offsetof(mrf_plan_desc, sigma),"
        " offsetof(mrf_plan_desc, stream), offsetof(mrf_plan_desc, batch_frames), sizeof(mrf_cg_info));return 0;}\n")
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(prog), "-o", str(exe)], check=True)
    vals = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()]
    D = binding.PlanDesc
    assert vals == [__import__("ctypes").sizeof(D), D.traj.offset, D.coils.offset, D.sigma.offset, D.stream.offset,
                    D.batch_frames.offset, __import__("ctypes").sizeof(binding.CGInfo)]


def test_status_strings(binding):
    for code, name in binding.STATUS.items():
        assert binding.lib.mrf_status_string(code).decode().startswith(name)


def _create(binding, **kw):
    import ctypes
    traj = kw.pop("traj", np.zeros((1, 4, 2), np.float32))
    d = binding.PlanDesc()
    d.N, d.L_local, d.frame_offset, d.M, d.R = kw.get("N", 32), kw.get("L", 2), 0, traj.shape[1], traj.shape[0]
    d.traj = traj.ctypes.data
    d.frame_interleaf = None
    d.C, d.coils = kw.get("C", 1), None
    d.W, d.sigma, d.flags = kw.get("W", 6), kw.get("sigma", 2.0), kw.get("flags", 0)
    d.device, d.stream, d.nccl_comm, d.batch_frames = 0, None, None, 0
    h = ctypes.c_void_p()
    return binding.lib.mrf_plan_create(ctypes.byref(d), ctypes.byref(h)), traj


@pytest.mark.parametrize("kw,code", [
    (dict(N=31), 1),                       # N odd
    (dict(N=6), 1),                        # N < 8
    (dict(L=0), 1),                        # L < 1
    (dict(W=1), 1), (dict(W=17), 1),       # W out of [2, 16]
    (dict(C=2), 1),                        # C > 1 without coils
    (dict(flags=8), 1),                    # unknown flag
    (dict(sigma=1.5), 5),                  # only sigma = 2
    (dict(N=40), 5),                       # G = 80 not a supported FFT size
    (dict(traj=np.full((1, 4, 2), 0.51, np.float32)), 1),    # |k| > 0.5
    (dict(traj=np.full((1, 4, 2), np.nan, np.float32)), 1),  # non-finite
])
def test_create_validation_codes(binding, kw, code):
    status, _ = _create(binding, **kw)
    assert status == code, binding.lib.mrf_last_error()
    assert binding.lib.mrf_last_error()


def test_null_arguments(binding):
    import ctypes
    assert binding.lib.mrf_plan_create(None, None) == 1
    assert binding.lib.mrf_forward(None, None, None, None) == 1
    assert binding.lib.mrf_adjoint(None, None, None, None) == 1
    assert binding.lib.mrf_normal(None, None, None, ctypes.c_float(0.0), None) == 1
    assert binding.lib.mrf_dc_cg(None, None, None, ctypes.c_float(0.0), 1, ctypes.c_float(0.0), None, None, None) == 1
    assert binding.lib.mrf_plan_destroy(None) == 1
    assert binding.lib.mrf_nccl_get_unique_id(None) == 1


def test_binding_fails_loudly_without_the_library(tmp_path):
    """The product path has no CPU fallback: importing the binding without libmrfnufft.so raises."""
    import shutil
    import subprocess
    import sys
    pkg = tmp_path / "paper_2310_05647_b200"
    pkg.mkdir()
    src = os.path.join(ROOT, "paper_2310_05647_b200")
    for name in ("__init__.py", "binding.py", "sharding.py"):
        if os.path.exists(os.path.join(src, name)):
            shutil.copy(os.path.join(src, name), pkg / name)
    code = "import paper_2310_05647_b200.binding"
    out = subprocess.run([sys.executable, "-c", code], cwd=tmp_path, capture_output=True, text=True)
    assert out.returncode != 0
    assert "ImportError" in out.stderr and "not built" in out.stderr
