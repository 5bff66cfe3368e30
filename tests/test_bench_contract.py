"""bench.py's JSON-line contract on CPU: the reference arm (the oracle, timed on the host) on the
smallest config prints one line with the keys the driver reads."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "1",
                          "--steps", "1", "--warmup", "0"], check=True, timeout=600, capture_output=True, text=True,
                         cwd=ROOT)
    lines = [ln for ln in out.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert "workload" in d["config"]


def test_reference_arm_config_and_clock():
    """Both arms print workload_config(); the reference arm's ms_per_step is its measured step
    wall time (what the driver's clock sees), the extrapolation is reported beside it."""
    sys.path.insert(0, ROOT)
    import argparse
    import bench
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "1",
                          "--steps", "1", "--warmup", "0"], check=True, timeout=600, capture_output=True, text=True,
                         cwd=ROOT)
    d = json.loads([ln for ln in out.stdout.strip().splitlines() if ln.startswith("{")][0])
    args = argparse.Namespace(config=1, exchange="allgather", bc="modify", tol=1e-10, deterministic=False,
                              method="fs")
    assert d["config"] == json.loads(json.dumps(bench.workload_config(args)))
    from fsfem_inputs import config_mesh, kuhn_counts
    c = kuhn_counts(*config_mesh(1).grid)
    assert d["config"]["n_faces"] == c["n_faces"] == 568 and d["config"]["nnz"] == 12879
    assert d["ms_per_step"] < 60e3 and d["extrapolated_ms_per_full_step"] > 0
