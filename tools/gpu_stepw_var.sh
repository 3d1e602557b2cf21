mkdir -p gpurun_out
L=$PWD/paper_2111_14317_b200
rm -f gpurun_out/swv.txt
PHT_STEPW=0 python tools/step_bench.py > gpurun_out/swv_tile.txt 2>&1; echo "tile $(tail -1 gpurun_out/swv_tile.txt)" >> gpurun_out/swv.txt
for v in lib lib_w8m2 lib_w4m5 lib_w2m8; do
  PHT_LIB=$L/$v/libpht.so python tools/step_bench.py > gpurun_out/swv_$v.txt 2>&1; echo "$v $(tail -1 gpurun_out/swv_$v.txt)" >> gpurun_out/swv.txt
done
