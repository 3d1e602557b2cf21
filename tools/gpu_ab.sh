set -x
PHT_LIB=$PWD/paper_2111_14317_b200/lib_rt/libpht.so python -m pytest tests -m gpu -q 2>&1 | tail -5 > gpurun_out/gpu_tests_rt.log
for v in lib lib_rt; do
  PHT_LIB=$PWD/paper_2111_14317_b200/$v/libpht.so python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_$v.json 2>gpurun_out/bench_$v.err
  PHT_LIB=$PWD/paper_2111_14317_b200/$v/libpht.so python tools/eval_bench.py > gpurun_out/eval_bench_$v.json 2> gpurun_out/eval_bench_$v.err
done
