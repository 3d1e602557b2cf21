mkdir -p gpurun_out
python -m pytest tests/test_gpu_fullsize.py -q > gpurun_out/full_tests.log 2>&1; echo "rc=$?" >> gpurun_out/full_tests.log
