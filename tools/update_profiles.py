"""Copies the evidence of one tools/gpu_profile.sh run from gpurun_out/ into profiles/ (tracked):
the default bench line, the ncu launch list summary, the ncu --set full summary and instruction
mix of one EMR step at the benched size (1000 x 512^2), and the per-kernel DRAM traffic that
bench.py reports as roofline.traffic -- with the algorithmic bytes of SURVEY §8(d) beside it
(the wasted-traffic ratio).

  python tools/update_profiles.py r02
"""
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT, PROF = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")
sys.path.insert(0, os.path.join(ROOT, "tools"))
import ncu_mix  # noqa: E402

PX = 1000 * 512 * 512                     # tools/prof_run.py --batch 1000 (config-2 images, EMR)
# the bench's kernel classes (bench.kernel_model names) and the launches of one step they cover
CLASSES = {"encode_kernel": ["encode_kernel"],
           "embed_prep+scan_kernel<embed>+finish": ["embed_prep_kernel", "scan_kernel<0, 1>", "scan_finish_kernel<0, 1>"],
           "scan_kernel<extract>+finish": ["scan_kernel<0, 0>", "scan_finish_kernel<0, 0>"],
           "recover_kernel+sse": ["recover_kernel"]}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def run(cmd):
    return subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT).stdout


def main(tag):
    sys.path.insert(0, ROOT)
    import bench

    line = json.loads([x for x in open(os.path.join(OUT, "bench_full.log")) if x.startswith("{")][-1])
    with open(os.path.join(PROF, f"{tag}_bench_default.json"), "w") as f:
        json.dump(line, f, indent=1)
    der = line["mean_der_bpp"]
    with open(os.path.join(PROF, f"{tag}_launches_emr.txt"), "w") as f:
        f.write(run([sys.executable, "tools/ncu_summary.py", "gpurun_out/launches_emr.csv"]))
    rep = os.path.join(OUT, "prof_all.ncu-rep")
    with open(os.path.join(PROF, f"{tag}_ncu_full_summary.txt"), "w") as f:
        f.write(f"# ncu --set full --clock-control none, one EMR step of tools/prof_run.py --batch 1000 "
                f"(config-2 images, {PX} px, inputs 4x the L2)\n")
        f.write(run([sys.executable, "tools/ncu_brief.py", rep]))
    rows = list(csv.reader(run(["ncu", "-i", rep, "--page", "raw", "--csv"]).splitlines()))
    hdr, units, data = rows[0], rows[1], rows[2:]
    idx = {h: i for i, h in enumerate(hdr)}

    def val(d, k):
        return float(d[idx[k]]) * SCALE.get(units[idx[k]], 1)

    per = {}
    for d in data:
        name = d[idx["Kernel Name"]]
        per.setdefault(name, []).append(d)
    mixf = open(os.path.join(PROF, f"{tag}_ncu_instruction_mix.txt"), "w")
    mixf.write("# executed-instruction mix per kernel (tools/ncu_mix.py: source page, one count per SASS address).\n"
               "# smsp__inst_executed.sum is the raw-page counter of the same capture; the source page comes from\n"
               "# another replay pass, so the two differ by the timing-dependent wait loops (SYNCS try_wait,\n"
               "# NANOSLEEP of the cross-CTA waits and their branches).\n")
    traffic, launches = {}, {}
    for cls, parts in CLASSES.items():
        rd = wr = dur = 0.0
        for part in parts:
            hits = [n for n in per if n.split("(")[0].split("::")[-1].replace("void ", "").strip().startswith(part)
                    or (part in n and "<" in part)]
            for n in hits:
                d = per[n][0]
                rd += val(d, "dram__bytes_read.sum")
                wr += val(d, "dram__bytes_write.sum")
                dur += float(d[idx["gpu__time_duration.sum"]])
                mixf.write(f"=== {n[:100]}\n    smsp__inst_executed.sum {float(d[idx['smsp__inst_executed.sum']]):.0f}\n")
                tot, alu, fma = 0, 0, 0
                import io
                import contextlib
                buf = io.StringIO()
                with contextlib.redirect_stdout(buf):
                    kname = part.split("<")[0]
                    skip = 1 if part in ("scan_kernel<0, 0>", "scan_finish_kernel<0, 0>") else 0
                    ncu_mix.main(rep, kname, 0, 10 ** 9, skip)
                mixf.write("    " + buf.getvalue().replace("\n", "\n    ").rstrip() + "\n")
                import re
                mm = re.search(r"total (\d+) warp-inst; alu-pipe (\d+) .*fma-pipe (\d+)", buf.getvalue())
                if mm:                                      # thread-instructions per pixel of the capture
                    t_, a_, f_ = (int(x) * 32 / PX for x in mm.groups())
                    mixf.write(f"    per pixel: {t_:.1f} thread-instructions, {a_:.1f} on the ALU pipe, {f_:.1f} on the FMA pipe\n")
        alg = bench.kernel_model(cls, der)["bytes"]
        traffic[cls] = (rd + wr) / PX
        launches[cls] = {"dram_read_bytes": rd, "dram_write_bytes": wr, "pixels": PX, "duration_us": dur,
                         "dram_bytes_per_px": (rd + wr) / PX, "algorithmic_bytes_per_px": alg,
                         "wasted_ratio": (rd + wr) / PX / alg if alg else None}
        d0 = per[[n for n in per if parts[0].split("<")[0] in n][0]][0]
        for k, kk in (("alu_pipe_pct", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
                      ("issue_active_pct", "smsp__issue_active.avg.pct_of_peak_sustained_active")):
            launches[cls][k] = float(d0[idx[kk]])
    mixf.close()
    old = {}
    try:
        old = json.load(open(os.path.join(PROF, "traffic.json")))
    except Exception:
        pass
    for k in ("coder_encode_kernel", "lmr_pack+header+coder_decode_kernels"):   # LMR coder entries (config 3)
        if k in old.get("bytes_per_px", {}):
            traffic[k] = old["bytes_per_px"][k]
            launches[k] = old["launches"][k]
    json.dump({"source": f"ncu --set full --clock-control none, one EMR step of tools/prof_run.py --batch 1000 "
                         f"(config-2 images, inputs 4x the L2), {tag}; per kernel class the DRAM bytes of its "
                         f"launches per pixel beside SURVEY 8(d)'s algorithmic bytes (d = {der:.3f}); the LMR "
                         f"coder entries are bytes per coded symbol (config 3, r01)",
               "bytes_per_px": traffic, "launches": launches},
              open(os.path.join(PROF, "traffic.json"), "w"), indent=1)
    for k, v in launches.items():
        if "wasted_ratio" in v:
            print(f"{k:40s} dram {v['dram_bytes_per_px']:.3f} B/px  algorithmic {v['algorithmic_bytes_per_px']:.3f}"
                  f"  ratio {v['wasted_ratio'] if v['wasted_ratio'] is None else round(v['wasted_ratio'], 3)}")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r02")
