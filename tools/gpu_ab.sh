mkdir -p gpurun_out
python -m pytest tests/test_gpu_proj.py -q > gpurun_out/proj_tests.log 2>&1; echo "rc=$?" >> gpurun_out/proj_tests.log
