"""bench.py plumbing on CPU: --gpus N starts N ranks (gloo dry run), the
reference arm honours --warmup and reports the same `config` object as our
arm (both built by bench.workload_config)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args, timeout=240):
    env = dict(os.environ, MASTER_ADDR="127.0.0.1")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                       capture_output=True, text=True, timeout=timeout, env=env)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout
    return json.loads(lines[0])


def test_gpus_2_starts_two_ranks():
    j = _run("--gpus", "2", "--dry-run")
    assert j["dry_run"] and j["n_gpus"] == 2 and j["ranks"] == [0, 1]
    assert j["config"]["workload"].startswith("C5")
    assert j["config"]["parallelism"].startswith("seq-split2")


def test_workload_config_is_shared_by_both_arms():
    sys.path.insert(0, ROOT)
    import bench
    assert bench.DEFAULT_WORKLOAD == "C5"
    for n in (1, 2, 4, 8):
        c = bench.workload_config("C5", n)
        assert c["global_batch"] == 1 and c["quantized_bytes_per_step"] == 142606336
    assert bench.workload_config("C2", 4)["global_batch"] == 32  # weak: a batch per GPU
    assert bench.workload_config("C3", 4)["global_batch"] == 32  # head shard: same job


def test_reference_arm_honours_warmup_and_config():
    from oracle import oracle as O
    if not O.have_ref():
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    sys.path.insert(0, ROOT)
    import bench
    j = _run("--impl", "reference", "--workload", "C1", "--steps", "3", "--warmup", "4")
    assert j["impl"] == "reference" and j["warmup"] == 4 and j["steps"] == 3
    assert j["config"] == bench.workload_config("C1", 1)
    assert j["cpu_baseline"]["kind"] == "reference" and j["e2e"]["h2d_bytes_per_step"] == 0


@pytest.mark.gpu
@pytest.mark.parametrize("workload,kind", [("C5", "seq-split2"), ("C3", "kv-head-shard2"), ("C2", "dp2")])
def test_two_rank_bench_on_one_gpu(workload, kind):
    """--gpus 2 end to end with both ranks on one GPU (BDK_BENCH_OVERSUB: gloo
    process group, rank r on GPU r % count): the sequence split with the
    peer-memory merge, the KV-head shard and the replicas run and report
    a whole-job line.  Timings of an oversubscribed GPU mean nothing."""
    env_prev = os.environ.get("BDK_BENCH_OVERSUB")
    os.environ["BDK_BENCH_OVERSUB"] = "1"
    try:
        j = _run("--gpus", "2", "--workload", workload, "--quick", "--no-cpu-baseline",
                 "--steps", "5", "--warmup", "3", "--e2e-steps", "2", "--soak", "0", timeout=600)
    finally:
        if env_prev is None:
            os.environ.pop("BDK_BENCH_OVERSUB", None)
        else:
            os.environ["BDK_BENCH_OVERSUB"] = env_prev
    assert j["n_gpus"] == 2 and j["value"] > 0 and j["gpu_launches"] > 0
    assert j["config"]["parallelism"].startswith(kind), j["config"]
