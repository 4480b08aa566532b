"""CPU checks of bench.py's bookkeeping (no GPU): the ncu evidence is used only while the
kernel sources it was captured on are unchanged, the oracle sample sizes are bounded, and the
reference arm's JSON line carries the contract's keys."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from synth.configs import CONFIGS  # noqa: E402


def test_src_sha_is_stable_and_source_keyed():
    a, b = bench.src_sha(), bench.src_sha()
    assert a == b and len(a) == 16


def test_ncu_evidence_requires_matching_sources(tmp_path, monkeypatch):
    d = tmp_path / "profiles" / "r02" / "ncu"
    d.mkdir(parents=True)
    (d / "traffic_pythia_scaled.json").write_text(json.dumps(
        {"kernel": "k", "dram_bytes_per_launch": 1.0, "src_sha": bench.src_sha()}))
    (d / "traffic_rho_scaled.json").write_text(json.dumps(
        {"kernel": "k", "dram_bytes_per_launch": 1.0, "src_sha": "0000000000000000"}))
    monkeypatch.setattr(bench, "ROOT", str(tmp_path))
    monkeypatch.setattr(bench, "src_sha", lambda: json.loads(
        (d / "traffic_pythia_scaled.json").read_text())["src_sha"])
    assert bench.ncu_evidence("pythia", "scaled")["dram_bytes_per_launch"] == 1.0
    assert bench.ncu_evidence("rho", "scaled") is None      # stale: captured on other sources
    assert bench.ncu_evidence("llama", "scaled") is None    # absent


def test_oracle_sample_is_bounded():
    for name, w in CONFIGS.items():
        n = bench.oracle_pairs_per_sample(w, 16)
        assert 1 <= n <= w.P
        assert n == 1 or n * 2 * w.T * w.V <= 2e7


def test_reference_arm_line():
    """--impl reference on the tiny config: one JSON line with the contract's keys."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--config", "tiny", "--steps", "1", "--warmup", "0"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "cpu_baseline", "e2e", "config"):
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "oracle"
