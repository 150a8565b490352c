#!/bin/bash
# one gpurun round trip for the evidence under profiles/: the default bench line (config 2 EMR,
# with the CPU-oracle baseline), an LMR line (config 3), the ncu launch list of the bench command
# (its device-resident steps only: --no-security --no-e2e, so the kernel shares compare with the line's)
# and one ncu --set full capture of the hot kernels (batch 128).
python bench.py > gpurun_out/bench_full.log 2>&1; echo bench=$?
python bench.py --config 3 --steps 10 --warmup 3 --cpu-seconds 10 > gpurun_out/bench_lmr.log 2>&1; echo bench_lmr=$?
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-security --no-e2e > gpurun_out/plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_emr.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-security --no-e2e > gpurun_out/ncu_launch.log 2>&1; echo ncu_launch=$?
python tools/prof_run.py --batch 128 --steps 2 > gpurun_out/prof_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on \
  -k regex:"encode_kernel|recover_kernel|scan_kernel|stats_kernel" -s 1 -c 5 -o gpurun_out/prof_all \
  python tools/prof_run.py --batch 128 --steps 2 > gpurun_out/prof_ncu.log 2>&1; echo ncu_full=$?
