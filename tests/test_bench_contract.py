"""bench.py's driver contract, on CPU: the reference arm's JSON line, rank handling under
torchrun, the host-thread count it reports, and the --gpus / WORLD_SIZE guard.  The GPU arm's
line is checked on the B200 by the round-end bench itself."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ARGS = ["--impl", "reference", "--config", "pubmed", "--steps", "1", "--warmup", "0",
        "--cpu-sample-edges", "2000"]


def _run(extra_env=None, args=ARGS):
    env = {k: v for k, v in os.environ.items()
           if k not in ("RANK", "LOCAL_RANK", "WORLD_SIZE", "OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS")}
    env.update(extra_env or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, env=env,
                          capture_output=True, text=True, timeout=300, cwd=ROOT)


def test_reference_arm_json_line():
    r = _run()
    assert r.returncode == 0, r.stderr
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 1 and d["steps"] == 1
    assert d["value"] > 0 and d["unit"] == "edges/s" and d["higher_is_better"] is True
    assert d["metric"].startswith("GCN epoch throughput")
    cb = d["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and "destination vertices" in cb["sample"]
    assert cb["nproc"] >= 1 and "tape_vs_port" in cb
    assert cb["value"] == d["value"]
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0
    assert d["config"]["workload"]


def test_reference_arm_under_torchrun_rank1_is_silent():
    r = _run({"RANK": "1", "LOCAL_RANK": "1", "WORLD_SIZE": "2"}, ARGS + ["--gpus", "2"])
    assert r.returncode == 0, r.stderr
    assert r.stdout.strip() == ""


def test_reference_arm_rank0_uses_all_host_threads():
    # torchrun exports OMP_NUM_THREADS=1 to every rank; the reference arm undoes it
    r = _run({"RANK": "0", "LOCAL_RANK": "0", "WORLD_SIZE": "2", "OMP_NUM_THREADS": "1"},
             ARGS + ["--gpus", "2"])
    assert r.returncode == 0, r.stderr
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["n_gpus"] == 2
    assert d["cpu_baseline"]["cores"] == len(os.sched_getaffinity(0))


def test_gpus_n_without_torchrun_self_launches_n_ranks():
    """``python bench.py --gpus 2`` (no WORLD_SIZE) re-launches itself under torch.distributed.run
    with 2 ranks on 127.0.0.1; rank 0 prints the one JSON line (the driver's scaling run may call
    either form)."""
    r = _run(args=ARGS + ["--gpus", "2"])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2


def test_gpus_mismatch_under_torchrun_is_refused():
    r = _run({"RANK": "0", "LOCAL_RANK": "0", "WORLD_SIZE": "3"}, ARGS + ["--gpus", "2"])
    assert r.returncode != 0
    assert "torch.distributed.run" in r.stderr
