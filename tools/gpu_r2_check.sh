#!/bin/bash
# Round-2 GPU check: the whole -m gpu suite, then a short bench run (one JSON line).
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/gpu_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/gpu_tests.log
tail -15 gpurun_out/gpu_tests.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?"
tail -c 1500 gpurun_out/bench.json
