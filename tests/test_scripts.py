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


def test_bench_roofline_fields():
    """bench.roofline() on synthetic per-kernel timings: the dominant kernel, its bound and
    fraction, and the coder's symbols/s against its issue floor."""
    sys.path.insert(0, ROOT)
    import bench
    peaks = {"hbm_gbs": 6556.2, "sm_max_mhz": 1965}
    HW = 512 * 512
    prof = {"encode_kernel": {"ms": 10.0, "launches": 20, "pixels": 20 * 1000 * HW},
            "coder_encode_kernel": {"ms": 30.0, "launches": 70, "pixels": 13_000_000_000},
            "lmr_pack+header+coder_decode_kernels": {"ms": 32.0, "launches": 30, "pixels": 10_400_000_000}}
    r = bench.roofline(prof, peaks, 1000, HW, [2.1 * HW] * 1000, "lmr")
    d = r["dominant"]
    assert d["kernel"] == "lmr_pack+header+coder_decode_kernels" and d["bound"] == "alu"
    assert abs(d["frac"] - d["achieved"] / d["peak"]) < 1e-12
    cs = d["coder_symbols"]
    assert abs(cs["achieved_sym_per_s"] - 10_400_000_000 / 0.032) < 1.0
    floor = 148 * 128 * 1965e6 / 39.0     # 4 SMSPs x 32 issue lanes per SM (224 tiles resident)
    assert abs(cs["issue_bound_sym_per_s"] - floor) < 1.0 and abs(cs["frac"] - cs["achieved_sym_per_s"] / floor) < 1e-12
    k = r["kernels"]["encode_kernel"]
    assert abs(k["algorithmic_GBps"] - 2.0 * 20 * 1000 * HW / 0.010 / 1e9) < 1e-6
    assert abs(sum(v["share"] for v in r["kernels"].values()) - 1.0) < 1e-12
