"""bench.py's driver contract on CPU: the reference arm's JSON line (config 1, the oracle port)
carries every key the driver reads, and both arms build `config` with the same function."""

import json
import subprocess
import sys
from types import SimpleNamespace

from conftest import ROOT

KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
        "scaling", "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"}


def test_reference_arm_line_contract():
    proc = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "mlp",
                           "--steps", "3", "--warmup", "1"], capture_output=True, text=True,
                          timeout=300, cwd=ROOT)
    assert proc.returncode == 0, proc.stderr[-2000:]
    lines = [ln for ln in proc.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert KEYS <= set(d), KEYS - set(d)
    assert d["impl"] == "reference" and d["steps"] == 3 and d["warmup"] == 1
    assert d["higher_is_better"] is True and d["value"] > 0
    cb = d["cpu_baseline"]
    assert {"value", "unit", "cores", "kind", "sample"} <= set(cb) and cb["kind"] == "port"
    assert cb["value"] == d["value"] and cb["cores"] >= 1
    assert {"schedule_spans_per_s", "run_crossover_job_iterations_per_s"} <= set(cb["reference_paths"])
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


def test_both_arms_share_the_config():
    sys.path.insert(0, str(ROOT))
    import bench

    for cfg, world in (("resnet50", 1), ("resnet50", 4), ("mlp", 1), ("mlp", 2)):
        args = SimpleNamespace(config=cfg, jobs=2, model="resnet50", batch=256, mix="", scenario="")
        a, b = bench.workload_config(args, world), bench.workload_config(args, world)
        assert a == b and a["parallelism"] == f"dp{world}"
        assert "workload" in a
