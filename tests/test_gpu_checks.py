"""Bounds-checked run of every kernel family (compute-sanitizer is closed on this
GPU pool, so the library has a checks build, -DMRF_CHECKS, in which every index read from a plan
table or a staged chunk -- gather records, spread cells and entries, chunk headers -- is tested
inside the kernels and a failure traps).  The small invocations of tools/sanitize_driver.py (all
G, both normal-operator forms, multi-batch / two-lane plans, a stress-like spiral with reduction
slices, CG / PCG, Phi_D, the MS-LLR step) must run through that build without a failed check."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


@pytest.mark.gpu
def test_bounds_checked_build_runs_clean():
    from paper_2310_05647_b200 import build
    lib = build.build(checks=True)   # in-tree; rebuilt only if a source is newer
    with open(lib, "rb") as f:
        assert b"MRF_CHECK failed" in f.read(), "the checks build carries no device checks"
    for dyn in ("", "1"):   # the plans' own choice of the k_adj_cols variant, then the dynamic one forced
        env = dict(os.environ, MRF_LIB_PATH=lib)
        if dyn:
            env["MRF_ADJ_DYN"] = dyn
        out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_driver.py"), "all" if not dyn else "ops"],
                             env=env, cwd=ROOT, capture_output=True, text=True, timeout=1500)
        log = out.stdout[-3000:] + out.stderr[-3000:]
        assert "MRF_CHECK failed" not in out.stdout + out.stderr, log
        assert out.returncode == 0, log
        tags = ["ops pr1 N=32 W=6", "ops mrf N=256 W=6", "ops cfg2 N=512 W=6", "ops pr1 N=32 W=2", "ops pr1 N=32 W=16",
                "ops stress N=128 W=8"] + ([] if dyn else ["dict: ok", "llr: ok"])
        for tag in tags:
            assert tag in out.stdout, log
