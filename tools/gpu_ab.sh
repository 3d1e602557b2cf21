mkdir -p gpurun_out
L=$PWD/paper_2111_14317_b200
for v in lib_old lib lib_m4 lib_old lib; do
  PHT_LIB=$L/$v/libpht.so python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1 --tracking "" --no-evaluation > gpurun_out/ab_bench_$v.json 2> gpurun_out/ab_bench_$v.err
  cat gpurun_out/ab_bench_$v.json >> gpurun_out/ab_all.jsonl
done
PHT_LIB=$L/lib/libpht.so python -m pytest tests -m gpu -q -x > gpurun_out/ab_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/ab_tests.log
