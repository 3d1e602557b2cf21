mkdir -p gpurun_out
L=$PWD/paper_2111_14317_b200
rm -f gpurun_out/ab_all.txt
for v in lib lib_gj lib_gjs lib_s; do
  PHT_LIB=$L/$v/libpht.so python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1 --tracking "" --no-evaluation > gpurun_out/ab_bench_$v.json 2> gpurun_out/ab_bench_$v.err
  echo "$v $(python -c "import json; print(json.load(open('gpurun_out/ab_bench_$v.json'))['value'])")" >> gpurun_out/ab_all.txt
  PHT_LIB=$L/$v/libpht.so python tools/track_bench.py katsura-10:10000 noon-10:10000 cyclic-10:1000000 > gpurun_out/ab_track_$v.txt 2>&1
  PHT_LIB=$L/$v/libpht.so python -m pytest tests/test_gpu_parity.py -q -x -k "pc_step or euler or evaluate_parity" > gpurun_out/ab_par_$v.log 2>&1; echo "$v parity rc=$?" >> gpurun_out/ab_all.txt
done
