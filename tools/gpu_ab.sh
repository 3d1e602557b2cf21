python -m pytest tests -m gpu -q 2>&1 | tail -8 > gpurun_out/gpu_tests.log
python tools/diag_cyclic10.py > gpurun_out/diag_c10.log 2>&1
python tools/track_bench.py katsura-10:10000 noon-10:10000 cyclic-10:1000000 > gpurun_out/tb.json 2>/dev/null
