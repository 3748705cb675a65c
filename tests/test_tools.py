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
