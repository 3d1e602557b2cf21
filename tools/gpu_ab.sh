for v in lib_d1 lib_d1w8 lib_d1w2; do
  PHT_LIB=$PWD/paper_2111_14317_b200/$v/libpht.so PHT_DENSE=1 python tools/eval_bench.py > gpurun_out/eb_$v.json 2>/dev/null
done
