"""The bench contract on CPU: the reference arm (`bench.py --impl reference`, the fp64 oracle
timed on host cores) prints one JSON line with the keys the driver reads, on the same metric
and config as the GPU arm; under torchrun only rank 0 prints."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env_extra=None):
    env = dict(os.environ)
    env.update(env_extra or {})
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       env=env, cwd=ROOT, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    return [ln for ln in r.stdout.splitlines() if ln.strip()]


def test_reference_arm_json_line():
    lines = _run(["--impl", "reference", "--steps", "1", "--warmup", "0", "--workload", "c1"])
    assert len(lines) == 1
    d = json.loads(lines[0])
    import bench
    assert d["impl"] == "reference" and d["metric"] == bench.METRIC and d["unit"] == bench.UNIT
    for k in ("value", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling", "vs_baseline",
              "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["value"] > 0 and d["higher_is_better"] is True and d["steps"] == 1
    assert d["config"]["workload"] == "c1"
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0
    # the GPU arm reports the same config (same function, same workload)
    import synth
    assert d["config"] == bench._config(synth.CONFIGS["c1"], 1)


def test_reference_arm_nonzero_rank_is_silent():
    lines = _run(["--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0", "--workload", "c1"],
                 {"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"})
    assert lines == []


def test_reference_arm_reports_n_gpus_and_its_config():
    """--gpus N without a launcher: the CPU arm reports n_gpus = N on the N-rank config (global
    batch N_loc * N), the same config the GPU arm reports at N ranks."""
    lines = _run(["--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0", "--workload", "c1"])
    d = json.loads(lines[0])
    import bench
    import synth
    assert d["n_gpus"] == 2 and d["config"] == bench._config(synth.CONFIGS["c1"], 2)
    assert d["config"]["global_batch"] == 2 * synth.CONFIGS["c1"].N_loc()
    host = d["cpu_baseline"]["host"]
    assert host["nproc"] >= 1 and host["lscpu_model"] and "governor" in host


def test_gpus_flag_launches_that_many_ranks():
    """`bench.py --gpus 2` outside torchrun re-launches itself as 2 ranks (torch.distributed.run,
    127.0.0.1); rank 0 alone prints.  --dry-run stops after the process group is up (gloo here,
    NCCL on a GPU box), so the launch path is checked without a GPU."""
    lines = _run(["--gpus", "2", "--dry-run"])
    assert len(lines) == 1, lines
    d = json.loads(lines[0])
    assert d["dry_run"] and d["n_gpus"] == 2 and d["ranks"] == [0, 1] and d["distinct_processes"] == 2


def test_world_size_must_match_gpus():
    env = dict(os.environ, RANK="0", WORLD_SIZE="2", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "4", "--dry-run"],
                       capture_output=True, text=True, env=env, cwd=ROOT, timeout=120)
    assert r.returncode != 0 and "refusing" in r.stderr


def test_roofline_peak_follows_the_clock():
    """the tensor roofline divides by the measured burst peak when the SM clock sat near
    its maximum during the timed region, by the sustained (power-capped) peak otherwise; both
    fractions and the step-level T_roof / T_step are always reported."""
    import bench
    import synth
    pk = {"hbm_gbs": 6546.6, "bf16_tflops": 1630.3, "bf16_tflops_sustained": 1378.5}
    cfg = synth.CONFIGS["c3"]
    args = (cfg, 1, 512, 535.0, 4.4e-3, 4.6)
    near = bench.roofline_block(*args, {"sm_mhz": 1940.0, "sm_max_mhz": 1965.0}, pk, 0.96)
    low = bench.roofline_block(*args, {"sm_mhz": 1450.0, "sm_max_mhz": 1965.0}, pk, 0.96)
    assert near["peak"] == 1630.3 and low["peak"] == 1378.5
    assert near["frac"] == near["frac_vs_burst"] and low["frac"] == low["frac_vs_sustained"]
    flops = 4.0 * 535.0 * cfg.C * 512
    assert abs(near["achieved"] - flops / 4.4e-3 / 1e12) < 1e-9
    st = near["step"]
    assert abs(st["t_roof_ms"] - flops / 1630.3e12 * 1e3) < 1e-9 and abs(st["frac"] - st["t_roof_ms"] / 4.6) < 1e-12
    assert near["executed_mma_flops_per_launch"] == 4.0 * (512 + 64) * cfg.C * 512   # 4 groups + a 64-row tail unit
    assert 0 < near["secondary"]["frac"] < 1
