"""Copies the evidence of one tools/gpu_profile.sh run from gpurun_out/ into profiles/ (tracked):
bench lines, the ncu launch list summary, the ncu --set full summary / instruction mix, and the
per-kernel dram traffic per pixel that bench.py reports as roofline.traffic.

  python tools/update_profiles.py r01
"""
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT, PROF = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")
NAME_MAP = {"encode_kernel": "encode_kernel", "recover_kernel": "recover_kernel",
            "scan_kernel<0, 1>": "embed_prep+scan_kernel<embed>+finish", "scan_kernel<0, 0>": "scan_kernel<extract>+finish",
            "stats_kernel": "stats_kernel"}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def run(cmd):
    return subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT).stdout


def main(tag):
    shutil.copy(os.path.join(OUT, "bench_full.log"), os.path.join(PROF, f"{tag}_bench_emr_config2.json"))
    shutil.copy(os.path.join(OUT, "bench_lmr.log"), os.path.join(PROF, f"{tag}_bench_lmr_config3.json"))
    with open(os.path.join(PROF, f"{tag}_launches_emr.txt"), "w") as f:
        f.write(run([sys.executable, "tools/ncu_summary.py", "gpurun_out/launches_emr.csv"]))
    rep = os.path.join(OUT, "prof_all.ncu-rep")
    with open(os.path.join(PROF, f"{tag}_ncu_full_summary.txt"), "w") as f:
        f.write(run([sys.executable, "tools/ncu_brief.py", rep]))
    with open(os.path.join(PROF, f"{tag}_ncu_instruction_mix.txt"), "w") as f:
        for k in ("encode_kernel", "recover_kernel", "scan_kernel"):
            f.write(f"=== {k} (first launch matching)\n")
            f.write(run([sys.executable, "tools/ncu_mix.py", rep, k]))
    rows = list(csv.reader(run(["ncu", "-i", rep, "--page", "raw", "--csv"]).splitlines()))
    hdr, units, data = rows[0], rows[1], rows[2:]
    idx = {h: i for i, h in enumerate(hdr)}
    px = 128 * 512 * 512                     # tools/prof_run.py --batch 128 (config-2 images)
    per_px, launches = {}, {}
    for d in data:
        key = [v for k, v in NAME_MAP.items() if k in d[idx["Kernel Name"]]]
        if not key:
            continue
        rd = float(d[idx["dram__bytes_read.sum"]]) * SCALE[units[idx["dram__bytes_read.sum"]]]
        wr = float(d[idx["dram__bytes_write.sum"]]) * SCALE[units[idx["dram__bytes_write.sum"]]]
        per_px[key[0]] = (rd + wr) / px
        launches[key[0]] = {"dram_read_bytes": rd, "dram_write_bytes": wr, "pixels": px,
                            "duration_us": float(d[idx["gpu__time_duration.sum"]]),
                            "alu_pipe_pct": float(d[idx["sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"]]),
                            "issue_active_pct": float(d[idx["smsp__issue_active.avg.pct_of_peak_sustained_active"]])}
    # LMR tile coder (units = coded symbols, as bench.py's profile counts them): wave 0 of an
    # encode (eta + candidate 0 of 1000 config-3 images, 16 tiles of 16384 symbols each) and one
    # decode (the map plane), from gpurun_out/prof_coder*.ncu-rep / prof_dec*.ncu-rep when present
    for name, pattern, syms in (("coder_encode_kernel", "prof_coder", 1000 * 2 * 16 * 16384),
                                ("lmr_pack+header+coder_decode_kernels", "prof_dec", 1000 * 16 * 16384)):
        reps = sorted((f for f in os.listdir(OUT) if f.startswith(pattern) and f.endswith(".ncu-rep")),
                      key=lambda f: os.path.getmtime(os.path.join(OUT, f)))
        if not reps:
            continue
        rr = list(csv.reader(run(["ncu", "-i", os.path.join(OUT, reps[-1]), "--page", "raw", "--csv"]).splitlines()))
        h2, u2, d2 = rr[0], rr[1], rr[2]
        i2 = {h: i for i, h in enumerate(h2)}
        rd = float(d2[i2["dram__bytes_read.sum"]]) * SCALE[u2[i2["dram__bytes_read.sum"]]]
        wr = float(d2[i2["dram__bytes_write.sum"]]) * SCALE[u2[i2["dram__bytes_write.sum"]]]
        per_px[name] = (rd + wr) / syms
        launches[name] = {"dram_read_bytes": rd, "dram_write_bytes": wr, "symbols": syms, "report": reps[-1],
                          "duration_us": float(d2[i2["gpu__time_duration.sum"]]),
                          "alu_pipe_pct": float(d2[i2["sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"]]),
                          "issue_active_pct": float(d2[i2["smsp__issue_active.avg.pct_of_peak_sustained_active"]])}
    json.dump({"source": f"ncu --set full --clock-control none, tools/prof_run.py --batch 128 (config-2 images, "
                         f"EMR), {tag}; cold-cache serialized replay: writes still resident in L2 at kernel end "
                         f"are not counted; the LMR coder entries are bytes per coded symbol (config 3)",
               "bytes_per_px": per_px, "launches": launches},
              open(os.path.join(PROF, "traffic.json"), "w"), indent=1)
    print(json.dumps(per_px, indent=1))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01")
