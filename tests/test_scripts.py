"""The driver-facing scripts at least compile (bench.py, __graft_entry__.py, tools/*.py), and
bench.py's argument parser accepts the driver's command line."""
import glob
import os
import py_compile
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_scripts_compile():
    files = [os.path.join(ROOT, "bench.py"), os.path.join(ROOT, "__graft_entry__.py")]
    files += glob.glob(os.path.join(ROOT, "tools", "*.py"))
    for f in files:
        py_compile.compile(f, doraise=True)


def test_bench_help_lists_the_driver_flags():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--help"], capture_output=True, text=True,
                         timeout=120).stdout
    for flag in ("--gpus", "--steps", "--warmup", "--impl", "--config", "--method"):
        assert flag in out
