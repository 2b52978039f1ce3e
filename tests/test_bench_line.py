"""bench.py keeps the driver's JSON-line contract: the GPU arm (small C1 run) and the reference arm
(the CPU oracle, no GPU needed) each print one line with the required keys."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout, env=None):
    env = dict(os.environ, RANK="0", WORLD_SIZE="1") if env is None else env
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, cwd=ROOT, capture_output=True,
                       text=True, timeout=timeout, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config", "e2e", "cpu_baseline"}


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--config", "C1", "--steps", "2", "--warmup", "1"], 600)
    assert BASE_KEYS <= d.keys()
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "queries/s"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["config"]["workload"].startswith("C1")


@pytest.mark.gpu
def test_gpu_arm_line():
    d = _run(["--config", "C1", "--steps", "3", "--warmup", "3", "--cpu-seconds", "2"], 900)
    assert BASE_KEYS <= d.keys() and "impl" not in d
    assert d["value"] > 0 and d["higher_is_better"] is True and d["scaling"] == "strong" and d["n_gpus"] == 1
    assert d["config"]["global_reads"] == d["config"]["reads_per_gpu"] == 11_000
    r = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= r.keys()
    assert r["bound"] == "hbm" and 0 < r["frac"] == pytest.approx(r["achieved"] / r["peak"])
    assert d["gpu_launches"] >= d["steps"]
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= d["clocks"].keys()
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["value"] > 0 and cb["extrapolated"] is True
    assert cb["single_thread"]["value"] > 0 and cb["all_cores"]["threads"] == cb["cores"]
    assert cb["agrees_with_gpu"] is True
    assert "random_access_roofline" in d
    # algorithmic bytes: at least the 8-byte read + 8-byte table pair + 8-byte result of a 32-bp read
    assert r["algorithmic_bytes_per_query"] >= 24


def _clean_env():
    return {k: v for k, v in os.environ.items()
            if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "LOCAL_WORLD_SIZE", "MASTER_ADDR", "MASTER_PORT")}


@pytest.mark.gpu
def test_gpu_arm_self_launches_two_ranks():
    """`--gpus 2` without torchrun starts 2 ranks (here sharing one GPU over gloo): strong scaling splits the
    job's Q reads into 2 contiguous shards, and the line reports n_gpus 2 with the whole job's reads."""
    d = _run(["--gpus", "2", "--dist-backend", "gloo", "--config", "C1", "--steps", "3", "--warmup", "3",
              "--no-cpu"], 900, env=_clean_env())
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert d["config"]["global_reads"] == 11_000 and d["config"]["reads_per_gpu"] == 5_500
    hits = sum(s[0] for s in d["shards"])
    assert len(d["shards"]) == 2 and hits > 0


def test_gpus_without_matching_world_size_fails():
    # a torchrun-style launch whose WORLD_SIZE disagrees with --gpus must not report a 1-GPU number
    env = dict(_clean_env(), RANK="0", WORLD_SIZE="1", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "8", "--config", "C1"], cwd=ROOT,
                       capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode != 0 and "WORLD_SIZE" in r.stderr
    assert not [ln for ln in r.stdout.splitlines() if ln.startswith("{")]


@pytest.mark.gpu
def test_partitioned_two_ranks_equal_replicated():
    """SURVEY.md 8(f) f4 end to end: `--partition` with 2 self-launched ranks (gloo, one GPU) exchanges the
    reads with real all-to-alls; the per-shard summaries (hits, sum of counts, checksum of every interval)
    equal those of the replicated index on the same reads."""
    import sys as _sys
    _sys.path.insert(0, ROOT)
    from paper_1303_3692_b200 import shard
    args = ["--gpus", "2", "--dist-backend", "gloo", "--config", "C2", "--steps", "3", "--warmup", "3", "--no-cpu",
            "--no-e2e", "--no-locate"]
    rep = _run(args, 900, env=_clean_env())
    part = _run(args + ["--partition"], 900, env=_clean_env())
    assert part["n_gpus"] == 2 and part["partition"]["nparts"] == 2
    assert shard.combine(part["shards"]) == shard.combine(rep["shards"])
