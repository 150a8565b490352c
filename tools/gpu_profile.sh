#!/bin/bash
# one gpurun round trip for the evidence under profiles/ (round tag $1, default r02):
#  1. the default bench line (config 2 EMR + the config-3 LMR block, CPU-oracle baselines);
#  2. the ncu launch list of the bench command's device-resident steps (--no-security --no-e2e,
#     so the kernel shares compare with the line's kernels block);
#  3. one ncu --set full capture of every kernel of one EMR step at the BENCHED size (1000 x 512^2,
#     inputs 4x the L2), so its dram bytes are the real per-launch traffic.
T=${1:-r02}
python bench.py > gpurun_out/bench_full.log 2>&1; echo bench=$?
python bench.py --config 2 --steps 2 --warmup 3 --no-cpu-baseline --no-security --no-e2e > gpurun_out/plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_emr.csv \
  python bench.py --config 2 --steps 2 --warmup 3 --no-cpu-baseline --no-security --no-e2e > gpurun_out/ncu_launch.log 2>&1; echo ncu_launch=$?
python tools/prof_run.py --batch 1000 --steps 2 > gpurun_out/prof_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on \
  -k regex:"encode_kernel|recover_kernel|scan_kernel|scan_finish|embed_prep" -s 8 -c 7 -o gpurun_out/prof_all \
  python tools/prof_run.py --batch 1000 --steps 2 > gpurun_out/prof_ncu.log 2>&1; echo ncu_full=$?
