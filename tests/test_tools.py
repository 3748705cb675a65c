"""The evidence tools run on the committed data (CPU only): the profiles report generator
and the tab:gentreesimu reproduction on a single-switch topology."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_profiles_report_generates():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "profiles_report.py")], capture_output=True,
                         text=True, cwd=ROOT, timeout=120)
    assert out.returncode == 0, out.stderr
    assert "## 1. bench.py lines" in out.stdout and "| 1 | 8 |" in out.stdout


def test_gentreesimu_tool_single_switch(tmp_path):
    dst = tmp_path / "g.json"
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "gentreesimu.py"), "--topos", "SS24",
                          "--out", str(dst)], capture_output=True, text=True, cwd=ROOT, timeout=300)
    assert out.returncode == 0, out.stderr
    d = json.load(open(dst))
    assert all(abs(r["rel_dev"]) < 0.05 for r in d["rows"])


def test_nvlcounters_summary():
    """Counter arithmetic used by bench.py's N > 1 roofline: exact byte counters preferred over
    the GPM rate estimate, per-direction bytes per step, nothing claimed when nothing moved."""
    sys.path.insert(0, ROOT)
    from tools.nvlcounters import summarize
    d = {"gpm_tx": 900, "gpm_rx": 800, "xmit_bytes": 2048, "rcv_bytes": 3072, "host_window_s": 1.0}
    s = summarize(d, 2, 1024)
    assert s["counters"] == "nvml xmit_bytes/rcv_bytes"
    assert (s["tx_bytes_per_step"], s["rx_bytes_per_step"]) == (1024, 1536)
    assert s["per_direction_vs_algorithmic"] == 1.5
    s = summarize({"gpm_tx": 4000, "gpm_rx": 2000, "xmit_bytes": 0, "rcv_bytes": 0}, 4, 1000)
    assert s["counters"] == "nvml gpm_tx/gpm_rx" and s["tx_bytes_per_step"] == 1000
    assert summarize({"host_window_s": 1.0}, 1, 1)["counters"] == "none answered"


def test_bench_reference_arm_line():
    """`bench.py --impl reference` (the CPU oracle as the reference arm) runs exactly the
    --steps K / --warmup W it is given and prints one JSON line with the contract's keys."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "2",
                          "--warmup", "1", "--cpu-sample-mib", "1"], capture_output=True, text=True, cwd=ROOT,
                         timeout=300)
    assert out.returncode == 0, out.stderr
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["steps"] == 2 and d["warmup"] == 1
    assert d["metric"] == "allreduce_busbw" and d["unit"] == "GB/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
