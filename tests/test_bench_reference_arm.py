"""CPU test of `bench.py --impl reference`: it prints the reference arm's
JSON line (oracle port on the host cores, same metric / config as the GPU
arm) and never maps the product library (libfse_b200.so)."""
import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_line_and_no_product_library():
    env = dict(os.environ, FSE_REF_SETTLE_S="0", CUDA_VISIBLE_DEVICES="")
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--impl", "reference", "--frames", "1",
                          "--steps", "1", "--warmup", "0"], capture_output=True, text=True, env=env,
                         cwd=REPO, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["metric"] == "lost_blocks_per_s"
    assert line["unit"] == "blocks/s" and line["higher_is_better"] is True
    assert line["value"] > 0 and line["e2e"]["value"] == line["value"]
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["config"]["workload"] == "config5" and line["config"]["blocks_per_step"] == 1620
    assert not any("libfse_b200" in p for p in line["native_libs_loaded"])
    assert any("liboracle" in p for p in line["native_libs_loaded"])
