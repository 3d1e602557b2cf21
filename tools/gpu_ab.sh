# A/B of the fused tensor-core row geometry (GeoD variants) vs scalar rows (PHT_DENSE=0)
mkdir -p gpurun_out
run() { # tag lib dense
  PHT_LIB=$2 PHT_DENSE=$3 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1 --tracking "" > gpurun_out/ab_bench_$1.json 2> gpurun_out/ab_bench_$1.err
  PHT_LIB=$2 PHT_DENSE=$3 python tools/track_bench.py katsura-10:10000 noon-10:10000 cyclic-10:1000000 > gpurun_out/ab_track_$1.txt 2>&1
}
L=$PWD/paper_2111_14317_b200
run scalar $L/lib/libpht.so 0
for v in gd32_2 gd16_2 gd16_3 gd32_1 gd8_4; do
  [ -f $L/lib_$v/libpht.so ] && run $v $L/lib_$v/libpht.so 1
done
PHT_LIB=$L/lib_gd16_2/libpht.so python -m pytest tests -m gpu -q -x > gpurun_out/ab_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/ab_tests.log
