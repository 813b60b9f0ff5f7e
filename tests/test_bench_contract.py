"""The bench.py JSON contract (the driver parses these lines): field names, types and the
relations between them, for the reference arm (CPU, the oracle) and for our arm (GPU)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
             "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config"}


def run_bench(*args, timeout=600):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                         capture_output=True, text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-3000:]
    return json.loads(lines[0])


def check_base(d, steps, warmup):
    assert BASE_KEYS <= set(d), BASE_KEYS - set(d)
    with open(os.path.join(ROOT, "BASELINE.json")) as f:
        assert d["metric"] == json.load(f)["metric"]
    assert d["unit"] == "GFLOP/s" and d["higher_is_better"] is True
    assert d["n_gpus"] == 1 and d["steps"] == steps and d["warmup"] == warmup >= 3
    assert d["value"] > 0 and d["ms_per_step"] > 0
    assert d["scaling"] in ("weak", "strong") and d["vs_baseline"] is None
    assert d["dtype"] == "f64" and d["data"] == "synthetic"
    assert isinstance(d["config"], dict) and "workload" in d["config"]
    e = d["e2e"]
    assert e["value"] > 0 and e["unit"] == d["unit"]
    assert e["h2d_bytes_per_step"] >= 0 and e["d2h_bytes_per_step"] >= 0


def test_reference_arm_contract():
    d = run_bench("--impl", "reference", "--steps", "1", "--warmup", "3")
    check_base(d, 1, 3)
    assert d["impl"] == "reference"
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"]
    assert cb["unit"] == d["unit"] and cb["sample"]
    assert d["e2e"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


@pytest.mark.gpu
def test_gpu_arm_contract():
    d = run_bench("--mesh", "30", "30", "30", "--steps", "2", "--warmup", "3",
                  "--no-cpu-baseline", "--no-format-compare")
    check_base(d, 2, 3)
    assert "impl" not in d or d["impl"] != "reference"
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s"
    assert r["achieved"] > 0 and r["peak"] > 0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-12
    assert "traffic" in r
    assert d["gpu_launches"] > 0
    a = d["assembly_roofline"]
    assert a["ms"] > 0 and a["bytes"] > 0 and abs(a["frac"] - a["achieved"] / a["peak"]) < 1e-12
    c = d["clocks"]
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(c)
    # the e2e number moves the step's inputs and the solution across the host boundary
    assert d["e2e"]["d2h_bytes_per_step"] >= 8 * 31 ** 3


def _bench_module():
    import importlib.util
    spec = importlib.util.spec_from_file_location("_bench", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


@pytest.mark.parametrize("gpus,env,mode,mesh", [
    (1, {}, "single", (300, 300, 300)),
    (2, {}, "multi", (600, 300, 300)),
    (4, {}, "multi", (600, 600, 300)),
    (8, {}, "multi", (600, 600, 600)),
    (1, {"WORLD_SIZE": "1", "RANK": "0", "LOCAL_RANK": "0"}, "rank", (300, 300, 300)),
    (8, {"WORLD_SIZE": "8", "RANK": "3", "LOCAL_RANK": "3"}, "rank", (600, 600, 600)),
])
def test_launch_forms(gpus, env, mode, mesh):
    """Both launch forms of `bench.py --gpus N` use N GPUs and say so: torchrun -> one RANK
    ctx per process; plain `--gpus N` -> one MULTI ctx over devices 0..N-1 (weak scaling,
    configs[4], by default)."""
    b = _bench_module()
    r = b.plan_run(gpus, "weak", env)
    assert r["mode"] == mode and r["n_gpus"] == gpus == r["world"]
    assert tuple(r["mesh"]) == mesh
    if mode == "multi":
        assert r["gpu_indices"] == list(range(gpus))
    if mode == "rank":
        assert r["rank"] == int(env["RANK"]) and r["gpu_indices"] == [int(env["LOCAL_RANK"])]
    s = b.plan_run(gpus, "strong", env)
    assert tuple(s["mesh"]) == (400, 400, 400) and s["n_gpus"] == gpus


def test_launch_form_errors():
    b = _bench_module()
    with pytest.raises(SystemExit):
        b.plan_run(2, "weak", {"WORLD_SIZE": "4"})          # --gpus must equal WORLD_SIZE
    with pytest.raises(SystemExit):
        b.plan_run(3, "weak", {})                           # weak scaling: 1/2/4/8 only
    assert b.plan_run(3, "strong", {})["mode"] == "multi"


def test_assembly_bytes_model():
    """SYM at 300^3: 14 value slots x 8 B + 9 run starts x 4 B + a 4 B mask per storage row
    (rows padded to 32) + b: the 4.36 GB per assembly VERDICT r01 measured against."""
    b = _bench_module()

    class Info:
        rows = local_rows = 301 ** 3
        sell_entries = 14 * 32 * ((301 ** 3 + 31) // 32)
    by = b.assembly_bytes(Info, "sym")
    assert abs(by / 1e9 - 4.36) < 0.01


@pytest.mark.gpu
def test_gpu_arm_under_torchrun_one_rank():
    """The torchrun launch form (RANK ctx, NCCL process group, uid broadcast) end to end at
    world size 1: same JSON contract, n_gpus 1."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=1",
           "--master-addr=127.0.0.1", "--master-port=29581", os.path.join(ROOT, "bench.py"),
           "--gpus", "1", "--mesh", "30", "30", "30", "--steps", "2", "--warmup", "3",
           "--no-cpu-baseline", "--no-format-compare"]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-3000:]
    d = json.loads(lines[0])
    check_base(d, 2, 3)
    assert "torchrun" in d["config"]["parallelism"]
