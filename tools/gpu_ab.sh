mkdir -p gpurun_out
L=$PWD/paper_2111_14317_b200
python -m pytest tests -m gpu -q -x > gpurun_out/ab_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/ab_tests.log
for v in lib lib_t256; do
  PHT_LIB=$L/$v/libpht.so python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1 --tracking "" > gpurun_out/ab_bench_$v.json 2> gpurun_out/ab_bench_$v.err
  PHT_LIB=$L/$v/libpht.so python tools/eval_bench.py > gpurun_out/ab_eval_$v.txt 2>&1
  PHT_LIB=$L/$v/libpht.so python tools/track_bench.py katsura-10:10000 noon-10:10000 cyclic-10:1000000 > gpurun_out/ab_track_$v.txt 2>&1
done
