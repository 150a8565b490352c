#!/bin/bash
# stability evidence: long runs (clocks sampled throughout) and three back-to-back default lines
python bench.py --config 2 --steps 2000 --warmup 10 --no-e2e --no-security --no-cpu-baseline > gpurun_out/sus_emr.log 2>&1; echo sus_emr=$?
python bench.py --config 3 --steps 200 --warmup 5 --no-e2e --no-security --no-cpu-baseline > gpurun_out/sus_lmr.log 2>&1; echo sus_lmr=$?
for i in 1 2 3; do python bench.py --cpu-seconds 5 > gpurun_out/rep$i.log 2>&1; echo rep$i=$?; done
