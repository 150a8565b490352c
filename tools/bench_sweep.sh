#!/bin/bash
# one gpurun round trip for the per-config bench lines under profiles/ (besides tools/gpu_profile.sh's
# default line): EMR and LMR configs 4 and 5, config 4 as one sharded job (--shard, strong-scaling
# mode; one rank here), config-1 latencies, the reduced-round cipher option at config 2 and the
# reference arm (the CPU oracle on the host cores).
python bench.py --config 4 --method emr --steps 5 --warmup 3 --no-cpu-baseline --no-security > gpurun_out/bench_emr_c4.log 2>&1; echo emr_c4=$?
python bench.py --config 5 --method emr --steps 5 --warmup 3 --no-cpu-baseline --no-security > gpurun_out/bench_emr_c5.log 2>&1; echo emr_c5=$?
python bench.py --config 4 --method lmr --steps 3 --warmup 3 --no-cpu-baseline --no-security > gpurun_out/bench_lmr_c4.log 2>&1; echo lmr_c4=$?
python bench.py --config 5 --method lmr --steps 3 --warmup 3 --no-cpu-baseline --no-security > gpurun_out/bench_lmr_c5.log 2>&1; echo lmr_c5=$?
python bench.py --config 4 --method emr --shard --steps 5 --warmup 3 --no-cpu-baseline --no-security --no-e2e > gpurun_out/bench_emr_c4_shard.log 2>&1; echo emr_c4_shard=$?
python bench.py --config 2 --cipher-rounds 12 --steps 50 --warmup 5 --no-cpu-baseline --no-security > gpurun_out/bench_emr_chacha12.log 2>&1; echo chacha12=$?
python bench.py --config 2 --cipher-rounds 8 --steps 50 --warmup 5 --no-cpu-baseline --no-security > gpurun_out/bench_emr_chacha8.log 2>&1; echo chacha8=$?
python tools/latency_config1.py --method emr > gpurun_out/lat_emr.log 2>&1; echo lat_emr=$?
python tools/latency_config1.py --method lmr > gpurun_out/lat_lmr.log 2>&1; echo lat_lmr=$?
python tools/both_keys_probe.py --config 2 > gpurun_out/both_emr.log 2>&1; echo both_emr=$?
python tools/both_keys_probe.py --config 3 > gpurun_out/both_lmr.log 2>&1; echo both_lmr=$?
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.log 2>&1; echo reference=$?
