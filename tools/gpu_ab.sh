mkdir -p gpurun_out
python -m pytest tests/test_gpu_edges.py -q > gpurun_out/edge_tests.log 2>&1; echo "rc=$?" >> gpurun_out/edge_tests.log
