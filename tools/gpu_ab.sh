python -m pytest tests -m gpu -q 2>&1 | tail -30 > gpurun_out/gpu_tests.log
python tools/diag_logstate.py > gpurun_out/diag.log 2>&1
