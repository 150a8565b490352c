#!/bin/bash
# one gpurun round trip for the per-config bench lines under profiles/ (besides tools/gpu_profile.sh's
# config 2 / config 3 lines): EMR configs 4 and 5, LMR configs 4 and 5, config-1 latencies.
python bench.py --config 4 --method emr --steps 5 --warmup 3 --no-cpu-baseline --no-security > gpurun_out/bench_emr_c4.log 2>&1; echo emr_c4=$?
python bench.py --config 5 --method emr --steps 5 --warmup 3 --no-cpu-baseline --no-security > gpurun_out/bench_emr_c5.log 2>&1; echo emr_c5=$?
python bench.py --config 4 --method lmr --steps 3 --warmup 3 --no-cpu-baseline --no-security > gpurun_out/bench_lmr_c4.log 2>&1; echo lmr_c4=$?
python bench.py --config 5 --method lmr --steps 3 --warmup 3 --no-cpu-baseline --no-security > gpurun_out/bench_lmr_c5.log 2>&1; echo lmr_c5=$?
python tools/latency_config1.py --method emr > gpurun_out/lat_emr.log 2>&1; echo lat_emr=$?
python tools/latency_config1.py --method lmr > gpurun_out/lat_lmr.log 2>&1; echo lat_lmr=$?
