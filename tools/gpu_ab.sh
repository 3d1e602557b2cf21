mkdir -p gpurun_out
rm -f gpurun_out/e2e.txt
for c in 8 16 32 64; do
  PHT_HOST_CHUNKS=$c python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 5 --tracking "" --no-evaluation > gpurun_out/e2e_$c.json 2>/dev/null
  echo "$c $(python -c "import json; d=json.load(open('gpurun_out/e2e_$c.json')); print(d['value'], d['e2e']['value'])")" >> gpurun_out/e2e.txt
done
