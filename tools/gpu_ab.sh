mkdir -p gpurun_out
python -m pytest tests/test_gpu_param.py -q -x > gpurun_out/param_tests.log 2>&1; echo "rc=$?" >> gpurun_out/param_tests.log
python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ab_bench.json 2> gpurun_out/ab_bench.err
python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1 --tracking "" --solver qr > gpurun_out/ab_bench_qr.json 2> gpurun_out/ab_bench_qr.err
python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1 --tracking "" --specialize > gpurun_out/ab_bench_spec.json 2> gpurun_out/ab_bench_spec.err
