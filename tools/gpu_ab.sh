mkdir -p gpurun_out
for i in 1 2; do python bench.py --no-cpu-baseline > gpurun_out/bench_v$i.json 2>/dev/null; done
PHT_HOST_CHUNKS=16 python bench.py --no-cpu-baseline --tracking "" --no-evaluation > gpurun_out/bench_c16.json 2>/dev/null
