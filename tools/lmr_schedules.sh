#!/bin/bash
# Tab. LMR_block_size shape on the synthetic corpus: config 3 (and config 4's LMR half) with rotation
# schedules {2^e..2^9}, e = 4 (paper default), 3, 2, 1 -> DER, good / bad cases, throughput.
for e in 4 3 2 1; do
  python bench.py --config 3 --lmr-emin $e --steps 3 --warmup 1 --no-cpu-baseline --no-security \
    > gpurun_out/lmr_sched_c3_e$e.log 2>&1; echo c3_e$e=$?
done
python bench.py --config 4 --method lmr --steps 2 --warmup 1 --no-cpu-baseline --no-security > gpurun_out/lmr_c4.log 2>&1; echo c4l=$?
python bench.py --config 4 --method emr --steps 5 --warmup 2 --no-cpu-baseline --no-security > gpurun_out/emr_c4.log 2>&1; echo c4e=$?
