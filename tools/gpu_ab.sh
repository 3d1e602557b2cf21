mkdir -p gpurun_out
L=$PWD/paper_2111_14317_b200
rm -f gpurun_out/evald_all.txt
for v in lib lib_m2w4 lib_m2w8; do
  echo "$v $(PHT_LIB=$L/$v/libpht.so python tools/eval_bench.py 2>/dev/null | tail -1)" >> gpurun_out/evald_all.txt
done
