#!/bin/bash
# one gpurun round trip for the LMR coder evidence (profiles/r02_ncu_lmr_coder.txt): ncu --set full
# of every tile-coder launch of one config-3 step (1000 x 512^2): the encode waves of the first
# encode call, then the loop's encode waves and the three decode calls (embed, extract: map plane;
# recover: eta + map), after the same command has exited 0 without ncu.
python tools/prof_run.py --config 3 --method lmr --batch 1000 --steps 1 > gpurun_out/lmr_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"coder_(en|de)code_fast" -c 17 \
  -o gpurun_out/prof_lmr_coder python tools/prof_run.py --config 3 --method lmr --batch 1000 --steps 1 \
  > gpurun_out/lmr_ncu.log 2>&1; echo ncu_lmr=$?
