# A/B of the warp-per-group step kernel (PHT_STEPW=1, default) vs the tile kernel (PHT_STEPW=0).
mkdir -p gpurun_out
rm -f gpurun_out/sw_all.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_edges.py -q -x -k "step or euler or pc" > gpurun_out/sw_tests.log 2>&1; echo "rc=$?" >> gpurun_out/sw_tests.log
for rep in 1 2; do
for m in 0 1; do
  PHT_STEPW=$m python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1 --tracking "" --no-evaluation > gpurun_out/sw_bench_$m.json 2> gpurun_out/sw_bench_$m.err
  echo "stepw=$m rep$rep $(python -c "import json; d=json.load(open('gpurun_out/sw_bench_$m.json')); print(round(d['value']/1e6,1), round(d['roofline']['frac'],4), round(d['e2e']['value']/1e6,1), {k: {p: round(v['points'][p]['graph_s']*1e3,3) for p in v['points']} for k, v in d['paper_protocol'].items()})")" >> gpurun_out/sw_all.txt
done
done
