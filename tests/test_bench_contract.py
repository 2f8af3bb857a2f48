"""bench.py keeps the driver's JSON contract (task spec): one JSON
line with the metric/config/timing keys, roofline, cpu_baseline, e2e, clocks,
gpu_launches, plus e2e_live, the configs[2]/[3] sub-lines and the configs[4]
validate_apply sweep; --impl reference prints the reference arm's line on the
identical configuration; --gpus N spawns N ranks.  Small step counts on the
BASELINE configs[1] shape (GPU); the rank spawn and plan line on CPU."""
import json
import os
import signal
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
# cfg3 needs > starvationK = 3 rounds: the first three are device-aborted by design
SMALL = ["--e2e-steps", "3", "--cpu-seconds", "0.5", "--live-rounds", "2", "--config-rounds", "5",
         "--cfg5-words-log2", "30", "--cfg5-log-mib", "16", "--cfg5-reps", "1"]


def _run(*extra, env=None, timeout=900):
    """bench.py in its own process group: on a timeout the whole group (the
    torchrun agent and every rank) is killed, so no rank outlives the test."""
    e = dict(os.environ)
    e.update(env or {})
    p = subprocess.Popen([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "3", "--warmup", "3", *extra],
                         stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True, cwd=ROOT, env=e,
                         start_new_session=True)
    try:
        stdout, stderr = p.communicate(timeout=timeout)
    except subprocess.TimeoutExpired:
        os.killpg(p.pid, signal.SIGKILL)
        p.communicate()
        raise
    assert p.returncode == 0, stderr[-3000:]
    lines = [ln for ln in stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, stdout[-2000:]
    return json.loads(lines[0])


@pytest.mark.gpu
def test_bench_line_has_the_contract_keys():
    d = _run(*SMALL)
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks",
              "e2e_live", "configs", "validate_apply"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["value"] > 0
    assert d["higher_is_better"] is True and d["scaling"] == "weak" and "workload" in d["config"]
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 1
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9 and r["traffic"]
    pf = r["protocol_floor"]  # the measured access-pattern floor of the same kernel
    assert pf["floor_kernel_ms"] > 0 and pf["kernel_over_floor"] > 1 and 0 < pf["dram_frac_of_peak"] < 1
    sb = d["step_breakdown_ms"]  # the device half of mergeCommit is inside the step
    assert sb["merge_stage"] > 0 and sb["batch"] > 0 and sb["validate_apply"] > 0
    assert d["shadow_equals_replica"] is True and d["bank_sum_ok"] is True
    c = d["cpu_baseline"]
    assert c["kind"] in ("port", "reference") and c["cores"] >= 1 and c["value"] > 0 and c["sample"]
    assert "full rounds" in c["sample"]
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert e["host_replica_matches_device"] is True
    lv = d["e2e_live"]
    assert "error" not in lv, lv
    assert lv["value"] > 0 and lv["dev_commits"] > 0 and lv["host_commits"] > 0 and lv["bank_sum_ok"] is True
    cf = d["configs"]
    assert cf["cfg3_zipf"]["value"] > 0 and cf["cfg4_cache"]["value"] > 0
    va = d["validate_apply"]
    assert va["n_gpus"] == 1 and va["gbs_algorithmic"] > 0 and va["sweep"][0]["entries_global"] > 0
    assert d["gpu_launches"] == 3 * sum(d["gpu_launches_per_step"].values())
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])


@pytest.mark.gpu
def test_reference_arm_line():
    d = _run("--impl", "reference")
    assert d["impl"] == "reference" and d["value"] > 0 and d["n_gpus"] == 1
    assert d["cpu_baseline"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0
    assert d["config"]["batch_tx"] == 1 << 20 and d["config"]["log_entries"] == 1 << 20  # identical config


@pytest.mark.gpu
def test_two_ranks_on_one_gpu():
    """--gpus 2 spawns two ranks (gloo, both on GPU 0): the multi-rank round
    with the fused NVLink-path router over CUDA IPC, and the sharded
    validate_apply sweep with its peer exchange."""
    d = _run("--gpus", "2", "--no-cpu-baseline", "--no-configs", "--live-rounds", "0", "--e2e-steps", "3",
             "--cfg5-reps", "1", env={"HETM_BENCH_BACKEND": "gloo", "HETM_BENCH_ONE_GPU": "1"})
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["bank_sum_ok"] is True
    va = d["validate_apply"]
    assert va["n_gpus"] == 2 and va["gbs_algorithmic"] > 0 and "NVLink" in va["exchange"]
    assert all(s["nvlink_bytes_out_per_rank"] > 0 for s in va["sweep"])


def test_plan_line_spawns_the_requested_ranks():
    """CPU: --gpus 2 outside torchrun re-launches under torch.distributed.run;
    both ranks join the process group (gloo) and the line reports n_gpus == 2
    with the configs[4] geometry and NVLink byte counts."""
    d = _run("--gpus", "2", "--plan", env={"HETM_BENCH_BACKEND": "gloo"}, timeout=300)
    assert d["plan"] is True and d["n_gpus"] == 2 and d["rank_count_checked"] == 2
    va = d["validate_apply"]
    assert va["shard_gib"] == 32.0 and va["stmr_gib_global"] == 64.0
    head = next(s for s in va["sizes"] if s["log_mib_global"] == 1024)
    assert head["entries_global"] == 2 * head["entries_ingested_per_rank"]
    assert head["nvlink_bytes_out_per_rank"] == head["entries_ingested_per_rank"] * 24 // 2


def test_plan_line_one_rank():
    d = _run("--plan", timeout=300)
    assert d["n_gpus"] == 1 and d["validate_apply"]["shard_gib"] == 64.0
    assert all(s["nvlink_bytes_total"] == 0 for s in d["validate_apply"]["sizes"])
