#!/bin/bash
# one gpurun round trip: GPU parity tests + a short bench (config 2 EMR); logs under gpurun_out/
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
python bench.py --steps 20 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench_emr.log 2>&1; echo bench=$?
