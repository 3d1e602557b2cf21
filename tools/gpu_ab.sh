mkdir -p gpurun_out
python -m pytest tests/test_gpu_proj.py -q > gpurun_out/proj_tests.log 2>&1; echo "rc=$?" >> gpurun_out/proj_tests.log
python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1 --tracking cyclic-10 > gpurun_out/ab_bench.json 2> gpurun_out/ab_bench.err
