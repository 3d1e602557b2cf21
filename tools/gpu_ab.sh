mkdir -p gpurun_out
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 --tracking "" --no-evaluation > gpurun_out/ab_bench.json 2> gpurun_out/ab_bench.err
