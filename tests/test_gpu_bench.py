"""bench.py contract on the GPU: one JSON line with the keys the driver reads; the multi-rank
path (torchrun, 2 ranks sharing the one GPU over gloo -- NCCL refuses duplicate GPUs) reports
the whole-job aggregate."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")


def _line(out):
    lines = [x for x in out.splitlines() if x.startswith("{")]
    assert len(lines) == 1, out[-2000:]
    return json.loads(lines[0])


def test_bench_single(gpu):
    r = subprocess.run([sys.executable, "bench.py", "--steps", "3", "--warmup", "3", "--instances", "50000",
                        "--no-e2e", "--no-baseline", "--no-secondary"], cwd=ROOT, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _line(r.stdout)
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "dtype", "config", "roofline", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["value"] > 0 and d["gpu_launches"] > 0
    assert d["roofline"]["bound"] == "alu" and 0 < d["roofline"]["frac"] < 1


def test_bench_two_ranks(gpu):
    """Config 5's multi-rank mode: a fixed total sharded over 2 ranks (strong scaling)."""
    env = dict(os.environ, FAR_BENCH_BACKEND="gloo")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", "29517", "bench.py", "--gpus", "2",
                        "--steps", "3", "--warmup", "3", "--instances", "20001", "--no-e2e", "--no-baseline",
                        "--no-secondary"], cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    d = _line(r.stdout)
    assert d["n_gpus"] == 2 and d["config"]["global_instances"] == 20001 and d["scaling"] == "strong"
    assert d["config"]["shard"] == [0, 10001]
    assert d["multi_gpu"]["allgather_ms_per_step_max_rank"] > 0


def test_bench_two_ranks_gathered_job_matches_oracle(gpu, O, tmp_path):
    """H9 end to end: bench.py's own strong-scaling step (shard_range shards, far_solve_many per rank,
    dist.gather_makespans + dist.gather_schedules) gathers the WHOLE job, in order, bit-exact
    against the oracle -- makespans and every task slot of every instance (ragged last shard)."""
    from paper_2507_13601_b200 import far, inputs
    total = 3001
    dump = str(tmp_path / "job.npz")
    env = dict(os.environ, FAR_BENCH_BACKEND="gloo")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", "29519", "bench.py", "--gpus", "2",
                        "--steps", "1", "--warmup", "3", "--instances", str(total), "--gather-schedules",
                        "--dump", dump, "--no-e2e", "--no-baseline", "--no-secondary"],
                       cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    import numpy as np
    job = np.load(dump)
    w = inputs.WORKLOADS["M5"]
    tab = w.table(count=total, parallel=True)
    ref, _ = O.far_many(w.profile, w.costs(), tab)
    assert job["makespan"].shape == (total,)
    assert (job["makespan"] == ref).all()
    slots = np.ascontiguousarray(job["slots"]).view(far.SLOT_DT)[..., 0]
    assert slots.shape == (total, w.n)
    for i in range(total):
        o = O.far(w.profile, w.costs(), tab[i])["slots"]
        assert (slots[i]["node"] == o["node"]).all() and (slots[i]["start"] == o["start"]).all(), i
        assert (slots[i]["size_used"] == o["size_used"]).all(), i
