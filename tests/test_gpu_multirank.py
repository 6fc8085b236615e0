"""Frame-sharded runs of the library with two live ranks (the
operator is block-diagonal over frames, so the only exchange is the sum over frames in the CG
inner products and in the LLR coefficient projection).

NCCL cannot put two ranks on one GPU, and every GPU run here has one device, so the two ranks
share cuda:0 and reduce through the plan's host hook (mrf_plan_set_host_allreduce -> gloo
all_reduce).  Everything else is the product path: each rank's plan covers its own frame block
(frame_offset, interleaf map), its CG scalars are the all-reduced partials, and the iterates must
equal the unsharded solve on one plan: per-frame operators are bit-deterministic, so only the
float64 summation order of the inner products differs.
"""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WORKER = os.path.join(ROOT, "tests", "multirank_worker.py")


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def run_ranks(mode: str, world: int, tmp_path):
    port = _free_port()
    procs = []
    for r in range(world):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, WORKER, mode, str(tmp_path)], env=env,
                                      stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True))
    outs = []
    for p in procs:
        try:
            o, _ = p.communicate(timeout=600)
        except subprocess.TimeoutExpired:
            p.kill()
            o, _ = p.communicate()
        outs.append(o)
    for p, o in zip(procs, outs):
        assert p.returncode == 0, o[-4000:]
    return [dict(np.load(os.path.join(tmp_path, f"rank{r}.npz"))) for r in range(world)]


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("cfg", ["mrf", "sense"])
def test_two_rank_cg_equals_unsharded(cfg, tmp_path):
    """mrf_dc_cg on 2 frame shards (host all-reduce of the fp64 CG scalars) = the unsharded solve:
    x to <= 1e-6, the residual history and the step lengths to <= 1e-12 (fp64 summation order)."""
    res = run_ranks(f"cg-{cfg}", 2, tmp_path)
    x = np.concatenate([r["x"] for r in res])
    ref = res[0]
    assert res[1]["offset"] == res[0]["x"].shape[0]
    assert rel(x, ref["x_full"]) <= 1e-6
    for r in res:                                   # every rank saw the same global scalars
        assert np.allclose(r["history"], ref["history_full"], rtol=1e-12, atol=0)
        assert np.allclose(r["alpha"], ref["alpha_full"], rtol=1e-12, atol=0)
    assert np.array_equal(res[0]["history"], res[1]["history"])


def test_two_rank_msllr_equals_unsharded(tmp_path):
    """Algorithm 1 (lambda_1 = 0, 4 iterations) on mrf_llr_create_shard operators over 2 frame
    shards: the [N^2][r] coefficient partials and the data-term partials are all-reduced; every
    rank holds identical maps; x and cost(n) match the unsharded solve (fp32 summation order of
    the coefficient projection)."""
    res = run_ranks("msllr", 2, tmp_path)
    x = np.concatenate([r["x"] for r in res])
    ref = res[0]
    assert rel(x, ref["x_full"]) <= 1e-5
    assert np.allclose(ref["cost"], ref["cost_full"], rtol=1e-5, atol=0)
    assert np.array_equal(res[0]["index"], res[1]["index"])
    assert np.mean(res[0]["index"] == ref["index_full"]) >= 0.999
