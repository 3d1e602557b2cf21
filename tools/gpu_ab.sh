# A/B of compile-time variants on one B200: step bench line, tracking times, step/eval parity.
# usage: bash tools/gpu_ab.sh lib lib_base ...   (directories under paper_2111_14317_b200/)
mkdir -p gpurun_out
L=$PWD/paper_2111_14317_b200
rm -f gpurun_out/ab_all.txt
for rep in 1 2; do
for v in "$@"; do
  PHT_LIB=$L/$v/libpht.so python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1 --tracking "" --no-evaluation --no-paper-protocol > gpurun_out/ab_bench_$v.json 2> gpurun_out/ab_bench_$v.err
  echo "$v rep$rep step $(python -c "import json; d=json.load(open('gpurun_out/ab_bench_$v.json')); print(round(d['value']/1e6,1), round(d['roofline']['frac'],4))")" >> gpurun_out/ab_all.txt
done
done
[ -n "$AB_FAST" ] && exit 0
for v in "$@"; do
  PHT_LIB=$L/$v/libpht.so python tools/track_bench.py katsura-10:10000 noon-10:10000 cyclic-10:1000000 > gpurun_out/ab_track_$v.txt 2>&1
  PHT_LIB=$L/$v/libpht.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_track.py -q -x > gpurun_out/ab_par_$v.log 2>&1; echo "$v parity rc=$?" >> gpurun_out/ab_all.txt
done
