# A/B: step bench line + standalone evaluation (generic/DMMA/specialised) for two library builds.
mkdir -p gpurun_out
L=$PWD/paper_2111_14317_b200
rm -f gpurun_out/ab2_all.txt
for rep in 1 2; do
for v in "$@"; do
  PHT_LIB=$L/$v/libpht.so python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1 --tracking "" --no-evaluation > gpurun_out/ab2_bench_$v.json 2> gpurun_out/ab2_bench_$v.err
  echo "$v rep$rep $(python -c "import json; d=json.load(open('gpurun_out/ab2_bench_$v.json')); print(round(d['value']/1e6,1), round(d['roofline']['frac'],4), {k: {p: round(v['points'][p]['graph_s']*1e3,3) for p in v['points']} for k, v in d['paper_protocol'].items()})")" >> gpurun_out/ab2_all.txt
done
done
for v in "$@"; do
  for m in 0 1; do PHT_DENSE=$m PHT_LIB=$L/$v/libpht.so python tools/eval_bench.py > gpurun_out/ab2_ev_${v}_$m.txt 2>&1; done
  PHT_SPEC=1 PHT_LIB=$L/$v/libpht.so python tools/eval_bench.py > gpurun_out/ab2_ev_${v}_spec.txt 2>&1
done
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/ab2_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ab2_tests.log
