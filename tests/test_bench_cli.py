"""bench.py's driver contract on CPU: `--gpus N` outside torchrun starts N
ranks itself (RANK / LOCAL_RANK / WORLD_SIZE set), and the reference arm runs
the CPU oracle without loading the product library, printing the same config
dict as the product arm would."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _json_lines(out: str):
    """Every JSON object in the output (ranks may write concurrently)."""
    dec = json.JSONDecoder()
    objs, i = [], out.find("{")
    while i >= 0:
        try:
            o, end = dec.raw_decode(out, i)
            objs.append(o)
            i = out.find("{", end)
        except json.JSONDecodeError:
            i = out.find("{", i + 1)
    return objs


@pytest.mark.timeout(300)
def test_gpus_2_spawns_two_ranks():
    env = dict(os.environ)
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--spawn-check"],
                       capture_output=True, text=True, env=env, timeout=280)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _json_lines(r.stdout)
    assert sorted(x["rank"] for x in lines) == [0, 1]
    assert sorted(x["local_rank"] for x in lines) == [0, 1]
    assert all(x["world"] == 2 and x["gpus"] == 2 for x in lines)


@pytest.mark.timeout(300)
def test_gpus_1_runs_in_process():
    env = dict(os.environ)
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK"):
        env.pop(k, None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "1", "--spawn-check"],
                       capture_output=True, text=True, env=env, timeout=280)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _json_lines(r.stdout)
    assert lines == [{"rank": 0, "world": 1, "local_rank": 0, "gpus": 1}]


def test_nccl_debug_summary(tmp_path):
    """Multi-rank lines carry NCCL's own account of the communicator (NCCL_DEBUG=INFO to a file)."""
    sys.path.insert(0, ROOT)
    import bench

    log = tmp_path / "nccl.log"
    log.write_text("host:1:1 [0] NCCL INFO NCCL version 2.28.9+cuda12.8\n"
                   "host:1:1 [0] NCCL INFO comm 0x1 rank 0 nRanks 8 nNodes 1 localRanks 8 localRank 0 MNNVL 0\n"
                   "host:1:1 [0] NCCL INFO NVLS multicast support is available on dev 0\n"
                   "host:1:1 [0] NCCL INFO Channel 00/0 : 0[0] -> 1[1] via P2P/CUMEM\n")
    out = bench.nccl_summary(str(log), 8)
    assert out["version"].startswith("2.28.9") and out["nvls"] and out["p2p_nvlink"] and out["ranks"] == 8
    assert bench.nccl_summary(None, 1) is None


@pytest.mark.timeout(600)
def test_reference_arm_is_independent_of_the_product_library():
    env = dict(os.environ)
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK"):
        env.pop(k, None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "c1",
                        "--steps", "1", "--warmup", "0", "--points", "300000"],
                       capture_output=True, text=True, env=env, timeout=580)
    assert r.returncode == 0, r.stderr[-2000:]
    (line,) = _json_lines(r.stdout)
    assert line["impl"] == "reference"
    assert not any("librasterbound" in p for p in line["libs_loaded"]), line["libs_loaded"]
    assert any("librb_oracle" in p for p in line["libs_loaded"])
    assert line["cpu_baseline"]["cpu_model"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0

    sys.path.insert(0, ROOT)
    import bench

    a = bench.parse(["--config", "c1", "--points", "300000"])
    w = bench.workload("c1", 300000, 0)
    assert line["config"] == json.loads(json.dumps(bench.config_dict(a, w, line["config"]["grid"]["max_level"], 1)))
